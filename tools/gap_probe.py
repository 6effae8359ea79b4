"""GPU idle gaps inside one Gotcha frame: torch.profiler (CUPTI) kernel and
memcpy activity of process_frame_device, gaps between consecutive activities."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1604_03622_b200 as kst  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 2001
cube = torch.from_numpy(scenes.bench_scene(3, q, q, seed=17).data[0]).cuda()
dop, grid = kst.make_doppler_grid(q), kst.make_spatial_grid(3)
for _ in range(3):
    kst.process_frame_device(cube, 1, 3, dop, grid)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        kst.process_frame_device(cube, 1, 3, dop, grid)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
half = len(evs) // 2
evs = evs[half:]  # second frame
t0 = evs[0].time_range.start
tot_busy = 0.0
gaps = []
prev_end = evs[0].time_range.start
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    if st > prev_end:
        gaps.append((st - prev_end, e.name[:50]))
    prev_end = max(prev_end, en)
    tot_busy += en - st
span = prev_end - t0
print(f"frame span {span:.1f} us, busy {tot_busy:.1f} us, idle {sum(g for g, _ in gaps):.1f} us in {len(gaps)} gaps")
for g, n in sorted(gaps, reverse=True)[:15]:
    print(f"  gap {g:7.1f} us before {n}")

import collections  # noqa: E402
agg = collections.OrderedDict()
for e in evs:
    nm = e.name
    for tag in ("kernel", "Kernel"):
        pass
    key = nm.split("(")[0].split("<")[0].split("::")[-1][:40]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.end - e.time_range.start
print("warm per-kernel (us):")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:24]:
    print(f"  {k:42s} {c:3d} {v:9.1f}")
