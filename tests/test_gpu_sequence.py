"""configs[2] on the GPU: parallel.process_sequence (frame sharding with the
upload/compute overlap) against per-frame oracle maps, in-process and under
torchrun with the NCCL map all-gather (world size 1 on the single-GPU box;
the N > 1 frame assignment and gather are covered by the gloo tests)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, map_tolerance, tight_tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import parallel, scenes  # noqa: E402

Q, G = 256, 16


def _frames(k):
    return [scenes.bench_scene(3, Q, Q, seed=1000 + f, movers=2).data[0] for f in range(k)]


def _oracle_maps(frames):
    out = []
    for fr in frames:
        ref = orc.pipeline(fr, 1, 3, Q, G)[3]
        m0 = orc.detect("kron", None, None, fr, orc.doppler_grid(Q), orc.spatial_grid(3, G)).max()
        out.append((ref, m0))
    return out


def test_process_sequence_mixed_inputs_match_oracle():
    frames = _frames(4)
    inputs = [frames[0], torch.from_numpy(frames[1]).pin_memory(),
              torch.from_numpy(frames[2]).cuda(), torch.from_numpy(frames[3])]
    maps = parallel.process_sequence(inputs, 1, 3, kst.make_doppler_grid(Q),
                                     kst.make_spatial_grid(3, G))
    assert tuple(maps.shape) == (4, Q, Q) and maps.is_cuda
    got = maps.cpu().numpy()
    for k, (ref, m0) in enumerate(_oracle_maps(frames)):
        err = np.abs(got[k] - ref)
        assert np.all(err <= map_tolerance(ref, m0))
        assert np.all(err <= tight_tolerance(ref, m0, "f32")), f"frame {k}"  # default precision


def test_process_sequence_torchrun_nccl_gather(tmp_path):
    out = tmp_path / "maps.npy"
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(ROOT, "tests", "helpers", "seq_nccl.py"), str(out), "3", str(Q)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "nranks 1" in r.stdout + r.stderr  # NCCL communicator came up (INIT log)
    got = np.load(out)
    assert got.shape == (3, Q, Q)
    for k, (ref, m0) in enumerate(_oracle_maps(_frames(3))):
        assert np.all(np.abs(got[k] - ref) <= tight_tolerance(ref, m0, "f32"))
