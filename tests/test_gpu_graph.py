"""FrameGraph: one frame of the fused pipeline captured as a CUDA graph
(kst_pipeline_async) and replayed per frame. Replays equal kst_pipeline
bitwise; frames outside the sync-free assumptions fall back to the
synchronous path; the graph is re-captured when resident device state
changes (kst_state_epoch)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1604_03622_b200 as kst  # noqa: E402
from paper_1604_03622_b200 import scenes  # noqa: E402
from paper_1604_03622_b200 import _native as nat  # noqa: E402
from oracle import kron_oracle as orc  # noqa: E402


def frames(p, q, n, k, seed=3):
    return [scenes.bench_scene(p, q, n, seed=seed + i, movers=2).data[0] for i in range(k)]


@pytest.mark.parametrize("p,q,n", [(3, 96, 40), (2, 251, 120), (4, 130, 65)])
def test_graph_replays_equal_pipeline(p, q, n):
    D, G = q, 16
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    cubes = frames(p, q, n, 3)
    buf = torch.empty((n, p, q), dtype=torch.complex128, device="cuda")
    fg = kst.FrameGraph(buf, 1, 3, dopplers=dop, spatial_grid=grid)
    fell_back = False
    for cube in cubes:
        buf.copy_(torch.from_numpy(cube))
        fg.replay()
        fell_back |= float(fg.rec[0]) != 1.0
        vals, summ = fg.result()
        ref, rsum = kst.process_frame_device(torch.from_numpy(cube).cuda(), 1, 3, dopplers=dop,
                                             spatial_grid=grid)
        assert torch.equal(vals, ref)
        assert np.array_equal(summ[:5], rsum[:5])
    # one capture serves every frame; a synchronous fallback may allocate its
    # own workspaces once (epoch change) and cost one re-capture
    assert fg.captures == 1 or (fell_back and fg.captures == 2)
    # against the oracle (the §8c tolerance of the headline path)
    fit, ua, ub, oref = orc.pipeline(cubes[-1], 1, 3, D, G)
    m0 = orc.detect("kron", None, None, cubes[-1], orc.doppler_grid(D), orc.spatial_grid(p, G)).max()
    v = vals[0].cpu().numpy()
    assert np.all(np.abs(v - oref) <= 1e-5 * np.abs(oref) + 1e-6 * m0)
    assert int(summ[0]) == fit.iterations


def test_graph_falls_back_and_recaptures():
    """A replayed frame whose device checks fail (k_B < r_B, all-zero) is
    recomputed by the synchronous path; work on another shape in between
    (constant banks, workspaces, detection tables change) forces a
    re-capture, and the results stay equal to kst_pipeline."""
    p, q, n, D, G = 3, 96, 40, 96, 16
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    base = frames(p, q, n, 1, seed=5)[0]
    buf = torch.empty((n, p, q), dtype=torch.complex128, device="cuda")
    fg = kst.FrameGraph(buf, 1, 3, dopplers=dop, spatial_grid=grid)

    def check(cube):
        buf.copy_(torch.from_numpy(cube))
        fg.replay()
        vals, summ = fg.result()
        ref, rsum = kst.process_frame_device(torch.from_numpy(cube).cuda(), 1, 3, dopplers=dop,
                                             spatial_grid=grid)
        assert torch.equal(vals, ref) and np.array_equal(summ[:5], rsum[:5])
        return summ

    check(base)
    one_bin = np.zeros_like(base)
    one_bin[0] = base[0]  # b of rank 1 < r_b: kb < 3 (device check fails -> sync path)
    s = check(one_bin)
    assert s[3] < 3
    s = check(np.zeros_like(base))  # zero estimate, identity filter
    assert s[0] == 0 and s[3] == 0
    e0 = nat.lib().kst_state_epoch()
    other = frames(2, 251, 60, 1, seed=11)[0]  # another shape on the same context
    kst.process_frame(other, 1, 3)
    assert nat.lib().kst_state_epoch() != e0
    c0 = fg.captures
    check(base)
    assert fg.captures == c0 + 1


def test_pipeline_async_rejects_ineligible_shapes():
    """kst_pipeline_async enqueues nothing outside the sync-free form."""
    buf = torch.zeros((8, 3, 32), dtype=torch.complex128, device="cuda")  # q <= 64
    fg = kst.FrameGraph(buf, 1, 3)
    with pytest.raises(kst.DimensionError):
        fg.replay()


@pytest.mark.parametrize("kind,groups", [("classical", 1), ("kron", 2), ("classical", 2)])
def test_graph_other_kinds_and_groups(kind, groups):
    """Replays equal the direct call for the other filter kinds and for
    multi-group (stacked) detection maps."""
    p, q, n = 3, 130, 60
    D, G = q, 16
    dop, grid = kst.make_doppler_grid(D), kst.make_spatial_grid(p, G)
    cube = frames(p, q, n, 1, seed=21)[0]
    buf = torch.from_numpy(cube).cuda()
    ref, rsum = kst.process_frame_device(buf, 1, 3, dopplers=dop, spatial_grid=grid, kind=kind,
                                         groups=groups)
    fg = kst.FrameGraph(buf, 1, 3, dopplers=dop, spatial_grid=grid, kind=kind, groups=groups)
    fg.replay()
    vals, summ = fg.result()
    assert torch.equal(vals, ref) and np.array_equal(summ[:5], rsum[:5])
