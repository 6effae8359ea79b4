"""Compare K1 engines (FP64 DMMA vs int8 slices) on a Gotcha-scale frame: S error and time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1604_03622_b200 as kst
from paper_1604_03622_b200 import scenes, lrkron
q = int(sys.argv[1]) if len(sys.argv) > 1 else 2001
cube = torch.from_numpy(scenes.bench_scene(3, q, q, seed=17).data[0]).cuda()
n, p, q = cube.shape
snaps = kst.cube_to_snapshots(cube)
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): out = fn()
    e1.record(); torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps
lrkron.set_gram_engine("dmma")
ref, t = timed(lambda: kst.sample_covariance(snaps, p, q).matrix)
print(f"dmma: {t:.3f} ms")
dg = ref.diagonal().real
scale = torch.sqrt(dg[:, None] * dg[None, :])
for s in (4, 5, 6, 7, 8):
    lrkron.set_gram_engine("int8", s)
    S, t = timed(lambda: kst.sample_covariance(snaps, p, q).matrix)
    err = (S - ref).abs()
    herm = (S - S.conj().T).abs().max().item()
    print(f"int8 s={s}: {t:.3f} ms  max|dS|/sqrt(SaaSbb)={(err/scale).max().item():.2e}  "
          f"|dS|_F/|S|_F={(torch.linalg.norm(S-ref)/torch.linalg.norm(ref)).item():.2e}  herm={herm:.1e}")
    vals, info = kst.process_frame(cube, 1, 3)
    print("   pipeline", info)
