"""NEXT rows through the C ABI vs the oracle.  Equal-budget 3-point RANSAC baseline: the
sampled triples and every per-hypothesis count bit-exact, fits within the transform tolerance, the same
winner; point-cloud resolution (row 3) bit-exact.  Needs a B200: `pytest -m gpu`."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_compare import ROT_TOL_RAD, TRANS_TOL, rot_angle_rad

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def TR():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import TurboReg

    return TurboReg


@pytest.mark.parametrize("key,n,iters,seed", [("A", None, 500, 1), ("B", 2000, 2000, 7), ("D", 1500, 1000, 2**63 + 5),
                                              ("B", 5000, 2000, 99)])
def test_ransac_matches_oracle(TR, key, n, iters, seed):
    from paper_2507_01439_b200._binding import I_CLIQUES, I_HYPS

    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=4, n=n)
    nn = inst["src"].shape[0]
    tr = TR(cfg.tau, iters, 1, cfg.inlier_threshold, max_n=nn)
    res = tr.ransac(inst["src"], inst["dst"], iters, seed)
    ref = oracle.ransac(inst["src"], inst["dst"], iters, seed, cfg.inlier_threshold, trace=True)
    cl = tr.intermediate(0, I_CLIQUES)[:iters]
    hy = tr.intermediate(0, I_HYPS)[:iters]
    assert np.array_equal(cl[:, :3], ref["cliques"][:, :3])  # the same sampled triples, slot by slot
    flag = hy[:, 13].copy().view(np.int32)
    assert np.array_equal(flag != 0, ref["hyp_degenerate"] != 0)
    ok = flag == 0
    assert np.array_equal(hy[ok, 12].copy().view(np.int32), ref["hyp_count"][ok])  # counts bit-exact
    for k in np.nonzero(ok)[0][:200]:
        assert rot_angle_rad(hy[k, :9].reshape(3, 3), ref["hyp_R"][k]) <= ROT_TOL_RAD
        assert np.abs(hy[k, 9:12] - ref["hyp_t"][k]).max() <= TRANS_TOL
    assert res["status"] == ref["status"] == 0
    assert res["inlier_count"] == ref["inlier_count"]
    assert tuple(res["clique"]) == tuple(ref["clique"])
    assert res["hypotheses_evaluated"] == ref["hypotheses_evaluated"]
    assert res["num_cliques"] == iters and res["num_pivots"] == 0 and res["clique_weight"] == 0


def test_ransac_then_turboreg_on_one_context(TR):
    # the RANSAC path leaves the context usable for registration (and vice versa), seeds reproduce
    from tests.gpu_compare import compare_pair

    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=5, n=1500)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=1500)
    a = tr.ransac(inst["src"], inst["dst"], 2000, 42)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)
    b = tr.ransac(inst["src"], inst["dst"], 2000, 42)
    assert all(np.array_equal(np.asarray(a[k]), np.asarray(b[k])) for k in a)


def test_ransac_budget_is_checked(TR):
    from paper_2507_01439_b200._binding import TurboRegError

    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=0)
    tr = TR(cfg.tau, 10, 2, cfg.inlier_threshold, max_n=inst["src"].shape[0])
    with pytest.raises(TurboRegError):
        tr.ransac(inst["src"], inst["dst"], 21, 0)
    with pytest.raises(TurboRegError):
        tr.ransac(inst["src"], inst["dst"], 0, 0)
    assert tr.ransac(inst["src"], inst["dst"], 20, 0)["num_cliques"] == 20


# ------------------------------------------------------------------------------------ NEXT(3) resolution
@pytest.mark.parametrize("n,seed", [(2, 0), (3, 1), (1000, 2), (5000, 3), (32768, 4)])
def test_point_resolution_matches_oracle(TR, n, seed):
    rng = np.random.default_rng(seed)
    xyz = rng.uniform(-1.5, 1.5, size=(n, 3)).astype(np.float32)
    if n >= 1000:
        xyz[5] = xyz[17]  # a duplicate point: nearest distance 0
    tr = TR(0.012, 10, 2, 0.1, max_n=max(n, 3))
    got = tr.point_resolution(xyz)
    if n <= 5000:
        assert got == oracle.point_resolution(xyz)  # bit-exact (same float32 tree, same order statistic)
    else:  # n = 32768: the oracle's O(n^2) loop is slow; check the order statistic on sampled points
        spatial = pytest.importorskip("scipy.spatial")
        d, _ = spatial.cKDTree(xyz.astype(np.float64)).query(xyz.astype(np.float64), k=2)
        ref = np.sort(d[:, 1])[(n - 1) // 2]
        assert abs(got - ref) <= 4e-7 * ref
    import torch

    assert tr.point_resolution(torch.from_numpy(xyz).cuda()) == got  # device input


def test_point_resolution_errors(TR):
    from paper_2507_01439_b200._binding import TurboRegError

    tr = TR(0.012, 10, 2, 0.1, max_n=100)
    with pytest.raises(TurboRegError):
        tr.point_resolution(np.zeros((1, 3), np.float32))
    # a cloud larger than max_n is fine: point_resolution has its own buffers (coincident points: pr = 0)
    assert tr.point_resolution(np.zeros((101, 3), np.float32)) == 0.0
    bad = np.zeros((10, 3), np.float32)
    bad[3, 1] = np.nan
    with pytest.raises(TurboRegError):
        tr.point_resolution(bad)
