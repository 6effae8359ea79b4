"""configs[4] (SURVEY.md §8 cfg 5): 4-pass 3-channel stacks through the fused
pipeline (kst_pipeline, groups = K) -- against the oracle at mid sizes where
the CPU restatement finishes in seconds. The full 2001 x 2001 stack is
checked against the unmodified reference's own outputs in
tests/test_gpu_fullsize_ref.py."""

import numpy as np
import pytest

from conftest import map_tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1604_03622_b200 as kst  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402
from paper_1604_03622_b200.pipeline import process_frame_device  # noqa: E402

K, P, G, RB = 4, 3, 16, 3


def _stack(q, seed, movers):
    hist = scenes.bench_scene(P, q, q, seed=seed, movers=movers, n_passes=K)
    return np.ascontiguousarray(kst.stack_passes(hist).data)


@pytest.mark.parametrize("q", [64, 251])
def test_fused_multipass_matches_oracle(q):
    st = _stack(q, 17, 4)
    s = orc.scm(st.reshape(q, -1), K * P, q)
    fit = orc.lrkron(s, K * P, q, K, RB)
    ua, ub = orc.filter_bases(fit)
    want = np.stack(orc.pass_maps("kron", ua, ub, st, K, P, orc.doppler_grid(q), G))
    x = torch.from_numpy(st).cuda()
    vals, summ = process_frame_device(x, K, RB, kst.make_doppler_grid(q),
                                      kst.make_stacked_spatial_grid(P, K, G), groups=K)
    assert int(summ[0]) == fit.iterations and bool(summ[1]) == fit.converged
    m0 = orc.detect("kron", None, None, st, orc.doppler_grid(q), orc.spatial_grid(K * P, G)).max()
    got = vals.cpu().numpy()
    assert np.all(np.abs(got - want) <= map_tolerance(want, m0))
