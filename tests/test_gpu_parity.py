"""CUDA path vs oracle, element by element, through the C ABI (needs a B200: `pytest -m gpu`)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_compare import compare_pair, rot_angle_rad
from tests.helpers import py_triangles
from paper_2507_01439_b200._binding import I_STATE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tr_mod():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import TurboReg

    return TurboReg


def _run_single(TurboReg, cfg, n=None, pair=0, max_n=None):
    inst = synth.workload_instance(cfg, pair=pair, n=n)
    nn = inst["src"].shape[0]
    tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=max_n or nn, max_batch=1)
    res = tr.register(inst["src"], inst["dst"])
    return tr, inst, res


@pytest.mark.parametrize("key", ["A", "B", "C", "D"])
def test_configs_full_parity(tr_mod, key):
    cfg = synth.CONFIGS[key]
    tr, inst, res = _run_single(tr_mod, cfg)
    stats = compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)
    print(key, stats)
    assert res["status"] == 0
    assert synth.rotation_error_deg(res["R"], inst["R"]) < 5.0


@pytest.mark.parametrize("n", [3, 4, 31, 32, 33, 63, 65, 97, 1337, 2049])
def test_ragged_sizes(tr_mod, n):
    cfg = synth.CONFIGS["A"]
    tr, inst, res = _run_single(tr_mod, cfg, n=n, max_n=max(n, 100))
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("k1,k2", [(1, 1), (7, 3), (500, 8), (300, 9), (5000, 2)])
def test_budgets(tr_mod, k1, k2):
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=3)
    tr = tr_mod(cfg.tau, k1, k2, cfg.inlier_threshold, max_n=cfg.n)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, k1, k2, cfg.inlier_threshold, result=res)


def test_batch_mixed_sizes_and_statuses(tr_mod):
    cfg = synth.CONFIGS["A"]
    sizes = [500, 2, 333, 600, 77, 0, 500]
    insts, srcs, dsts = [], [], []
    for p, n in enumerate(sizes):
        inst = synth.workload_instance(cfg, pair=10 + p, n=max(n, 1))
        s, d = inst["src"][:n], inst["dst"][:n]
        if p == 6:
            d = d.copy()
            d[17, 1] = np.nan
        insts.append(inst)
        srcs.append(s)
        dsts.append(d)
    n = np.array(sizes, np.int32)
    off = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=550, max_batch=len(sizes))
    res = tr.register_batch(np.concatenate(srcs), np.concatenate(dsts), off, n)
    assert [int(r) for r in res["status"]] == [0, 2, 0, 3, 0, 2, 4]
    for p in (0, 2, 4):
        r = {k: res[p][k] for k in res.dtype.names}
        compare_pair(tr, p, srcs[p], dsts[p], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)
    for p in (1, 3, 5, 6):
        assert np.all(res[p]["R"] == 0) and np.all(res[p]["t"] == 0)


def test_batch_mixed_row_widths(tr_mod):
    # a pair above 256 words per row (n = 9000) gives the whole batch 256-entry sparse-row lists; the small
    # pair in the same batch must still match the oracle, and both must match their single-pair calls
    cfg = synth.CONFIGS["B"]
    big = synth.workload_instance(cfg, pair=40, n=9000)
    small = synth.workload_instance(cfg, pair=41, n=2500)
    n = np.array([2500, 9000], np.int32)
    off = np.array([0, 2500], np.int64)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=9000, max_batch=2)
    res = tr.register_batch(np.concatenate([small["src"], big["src"]]), np.concatenate([small["dst"], big["dst"]]),
                            off, n)
    assert [int(r) for r in res["status"]] == [0, 0]
    r = {k: res[0][k] for k in res.dtype.names}
    compare_pair(tr, 0, small["src"], small["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)
    one_small = tr.register(small["src"], small["dst"])
    one_big = tr.register(big["src"], big["dst"])
    for one, b in ((one_small, res[0]), (one_big, res[1])):
        assert tuple(one["clique"]) == tuple(b["clique"]) and one["inlier_count"] == b["inlier_count"]
        assert one["num_edges"] == b["num_edges"] and one["num_cliques"] == b["num_cliques"]


def test_device_inputs_match_host_inputs(tr_mod):
    import torch

    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=5)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=2)
    host = tr.register_batch(np.concatenate([inst["src"]] * 2), np.concatenate([inst["dst"]] * 2),
                             np.array([0, cfg.n]), np.array([cfg.n, cfg.n]))
    ds = torch.from_numpy(np.concatenate([inst["src"]] * 2)).cuda()
    dd = torch.from_numpy(np.concatenate([inst["dst"]] * 2)).cuda()
    out = torch.zeros(2 * 104, dtype=torch.uint8, device="cuda")
    tr.register_batch(ds, dd, np.array([0, cfg.n]), np.array([cfg.n, cfg.n]), out=out)
    torch.cuda.synchronize()
    from paper_2507_01439_b200 import RESULT_DTYPE

    dev = out.cpu().numpy().view(RESULT_DTYPE)
    assert dev.tobytes() == host.tobytes()
    assert host[0].tobytes() == host[1].tobytes()


@pytest.mark.parametrize("density", [0.05, 0.2, 0.5])
@pytest.mark.parametrize("seed", range(2))
def test_injected_adjacency_full_budget(tr_mod, density, seed):
    # SC^2 weights bit-exact and App. C: O2 with K1 = all edges, K2 = N gives every triangle exactly once
    n = 60 + 37 * seed
    C = synth.erdos_renyi(n, density, 900 + seed)
    tr = tr_mod(0.01, n * n, n, 0.1, max_n=n)
    tr.pgs_from_adjacency(C)
    from paper_2507_01439_b200._binding import I_CLIQUES, I_PIVOTS, I_SC2

    G = tr.intermediate(0, I_SC2)
    assert (G == oracle.sc2(C)).all()
    O = oracle.o2(oracle.sc2(C))
    piv = oracle.select_pivots(O, n * n)
    assert sorted(map(tuple, piv.tolist())) == sorted(map(tuple, tr.intermediate(0, I_PIVOTS).tolist()))
    cl = tr.intermediate(0, I_CLIQUES)
    cl = cl[cl[:, 0] >= 0]
    assert sorted(map(tuple, cl[:, :3].tolist())) == sorted(py_triangles(C))
    ref, _ = oracle.pgs(O, piv, n)
    assert sorted(map(tuple, cl.tolist())) == sorted(map(tuple, ref.tolist()))


@pytest.mark.parametrize("k1,k2", [(3, 2), (40, 1), (100, 5)])
def test_injected_adjacency_budgets(tr_mod, k1, k2):
    n = 150
    C = synth.erdos_renyi(n, 0.2, 4242)
    tr = tr_mod(0.01, k1, k2, 0.1, max_n=n)
    tr.pgs_from_adjacency(C)
    from paper_2507_01439_b200._binding import I_CLIQUES, I_PIVOTS

    O = oracle.o2(oracle.sc2(C))
    piv = oracle.select_pivots(O, k1)
    assert list(map(tuple, piv.tolist())) == list(map(tuple, tr.intermediate(0, I_PIVOTS).tolist()))
    ref, _ = oracle.pgs(O, piv, k2)
    cl = tr.intermediate(0, I_CLIQUES)
    cl = cl[cl[:, 0] >= 0]
    assert sorted(map(tuple, cl.tolist())) == sorted(map(tuple, ref.tolist()))


def test_complete_graph_all_ties(tr_mod):
    # K_N: every weight N-2, the K1 pivots are the lexicographically first edges
    n = 70
    C = (1 - np.eye(n)).astype(np.uint8)
    tr = tr_mod(0.01, 100, 3, 0.1, max_n=n)
    tr.pgs_from_adjacency(C)
    from paper_2507_01439_b200._binding import I_CLIQUES, I_PIVOTS

    piv = tr.intermediate(0, I_PIVOTS)
    lex = [(i, j) for i in range(n) for j in range(i + 1, n)][:100]
    assert list(map(tuple, piv[:, :2].tolist())) == lex and (piv[:, 2] == n - 2).all()  # (w desc, i, j) order
    cl = tr.intermediate(0, I_CLIQUES)
    O = oracle.o2(oracle.sc2(C))
    ref, _ = oracle.pgs(O, oracle.select_pivots(O, 100), 3)
    assert sorted(map(tuple, cl[cl[:, 0] >= 0].tolist())) == sorted(map(tuple, ref.tolist()))


@pytest.mark.parametrize("n,k1", [(70, 100), (200, 300), (200, 20000)])
def test_complete_graph_tie_paths(tr_mod, n, k1):
    # all weights tie: <= 8192 candidates use the candidate sort, more use the ordered count/scan/emit path;
    # both must pick the lexicographically first K1 edges
    C = (1 - np.eye(n)).astype(np.uint8)
    tr = tr_mod(0.01, k1, 2, 0.1, max_n=n)
    tr.pgs_from_adjacency(C)
    from paper_2507_01439_b200._binding import I_CLIQUES, I_PIVOTS

    piv = tr.intermediate(0, I_PIVOTS)
    lex = [(i, j) for i in range(n) for j in range(i + 1, n)][:k1]
    assert sorted(map(tuple, piv[:, :2].tolist())) == lex and (piv[:, 2] == n - 2).all()
    O = oracle.o2(oracle.sc2(C))
    ref, _ = oracle.pgs(O, oracle.select_pivots(O, k1), 2)
    cl = tr.intermediate(0, I_CLIQUES)
    assert sorted(map(tuple, cl[cl[:, 0] >= 0].tolist())) == sorted(map(tuple, ref.tolist()))


def test_tau_base_plane(tr_mod):
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=8)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, tau_base=4 * cfg.tau, max_n=cfg.n)
    res = tr.register(inst["src"], inst["dst"])
    Cb = tr.bits(0, base=True)
    ref_b, eb, _, _ = oracle.compat(inst["src"], inst["dst"], 4 * cfg.tau)
    assert (Cb == ref_b).all()
    from paper_2507_01439_b200._binding import I_STATE

    assert tr.intermediate(0, I_STATE)["edges_base"] == eb
    C = tr.bits(0)
    assert (C <= Cb).all()  # τ-monotonicity
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


def test_noise_free_exact_recovery(tr_mod):
    # App. A.3: congruent triangles fix T; 0 outliers, σ = 0 → every inlier counted
    inst = synth.generate(400, 1.0, (1, 1, 1), 0.0, seed=31)
    tr = tr_mod(0.001, 200, 2, 0.001, max_n=400)
    res = tr.register(inst["src"], inst["dst"])
    assert res["status"] == 0 and res["inlier_count"] == 400
    assert rot_angle_rad(res["R"], inst["R"]) < 1e-5
    assert np.abs(res["t"] - inst["t"]).max() < 1e-5


def test_no_hypothesis(tr_mod):
    # all-outlier, tiny τ: no edge has a positive SC^2 weight → NoHypothesis, zero transform
    rng = np.random.default_rng(0)
    src = rng.uniform(-1, 1, (300, 3)).astype(np.float32)
    dst = rng.uniform(-1, 1, (300, 3)).astype(np.float32)
    tr = tr_mod(1e-7, 100, 2, 0.01, max_n=300)
    res = tr.register(src, dst)
    assert res["status"] == 5 and np.all(res["R"] == 0) and res["num_pivots"] == 0


@pytest.mark.parametrize("case", ["triplicates", "one_point"])
def test_duplicate_points(tr_mod, case):
    # coincident correspondences: tests with S = 0 are never certified by the filter (S <= τ²(1 + 2^-16)), so
    # every lane meeting one redoes its tests with the exact tree; all-identical points give the complete
    # graph (|0 − 0| <= τ), all-tied weights and degenerate (non-unique) Kabsch fits
    cfg = synth.CONFIGS["B"]
    if case == "triplicates":
        inst = synth.workload_instance(cfg, pair=9, n=300)
        src = np.repeat(inst["src"], 3, axis=0)
        dst = np.repeat(inst["dst"], 3, axis=0)
        perm = np.random.default_rng(5).permutation(900)
        src, dst = src[perm], dst[perm]
    else:
        src = np.tile(np.array([[0.5, -0.25, 2.0]], np.float32), (150, 1))
        dst = np.tile(np.array([[-1.0, 0.75, 0.125]], np.float32), (150, 1))
    n = src.shape[0]
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n)
    res = tr.register(src, dst)
    compare_pair(tr, 0, src, dst, cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


def test_full_size_batch_sampled_parity(tr_mod):
    # BASELINE sizes in the bench's launch configuration (a batch of config-E pairs), sampled pairs checked
    # against the oracle element by element, every pair checked for planted recovery.
    cfg = synth.CONFIGS["E"]
    P = 6
    insts = [synth.workload_instance(cfg, pair=p) for p in range(P)]
    n = np.full(P, cfg.n, np.int32)
    off = (np.arange(P) * cfg.n).astype(np.int64)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=P)
    res = tr.register_batch(np.concatenate([i["src"] for i in insts]), np.concatenate([i["dst"] for i in insts]),
                            off, n)
    for p in (0, P - 1):
        r = {k: res[p][k] for k in res.dtype.names}
        compare_pair(tr, p, insts[p]["src"], insts[p]["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)
    for p in range(P):
        assert res[p]["status"] == 0
        assert synth.rotation_error_deg(res[p]["R"].reshape(3, 3), insts[p]["R"]) <= 5
        assert synth.translation_error(res[p]["t"], insts[p]["t"]) <= 0.1


@pytest.mark.parametrize("path,min_rows", [(0, 1), (0, 128), (1, 128), (2, 1)])
@pytest.mark.parametrize("key,n", [("A", None), ("B", 1500), ("D", 2100), ("C", None)])
def test_sc2_paths_agree_with_oracle(tr_mod, path, min_rows, key, n):
    # tensor-core dense block (path 0), popcount only (1), CUDA-core dp4a dense block (2): identical Ĝ
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=1, n=n)
    nn = inst["src"].shape[0]
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn)
    tr.set_option("sc2_path", path)
    tr.set_option("heavy_min_rows", min_rows)
    tr.set_option("heavy_min_degree", 1 if min_rows == 1 else 32)
    res = tr.register(inst["src"], inst["dst"])
    from paper_2507_01439_b200._binding import I_STATE

    st = tr.intermediate(0, I_STATE)
    if path == 1:
        assert st["heavy_h"] == 0
    elif min_rows == 1:
        assert st["heavy_h"] > 0
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


def test_sc2_heavy_block_on_dense_injected_graph(tr_mod):
    # a graph whose heavy block spans several 128×256 MMA tiles plus a ragged edge
    n = 900
    C = synth.erdos_renyi(n, 0.04, 77)
    rng = np.random.default_rng(1)
    dense = rng.choice(n, 700, replace=False)
    for a in dense:
        row = dense[rng.random(700) < 0.7]
        C[a, row] = 1
        C[row, a] = 1
    np.fill_diagonal(C, 0)
    tr = tr_mod(0.01, 500, 3, 0.1, max_n=n)
    tr.set_option("heavy_min_rows", 1)
    tr.pgs_from_adjacency(C)
    from paper_2507_01439_b200._binding import I_CLIQUES, I_SC2, I_STATE

    assert tr.intermediate(0, I_STATE)["heavy_h"] > 256
    assert (tr.intermediate(0, I_SC2) == oracle.sc2(C)).all()
    O = oracle.o2(oracle.sc2(C))
    ref, _ = oracle.pgs(O, oracle.select_pivots(O, 500), 3)
    cl = tr.intermediate(0, I_CLIQUES)
    assert sorted(map(tuple, cl[cl[:, 0] >= 0].tolist())) == sorted(map(tuple, ref.tolist()))


@pytest.mark.parametrize("scale,tau", [(1.5, 0.5), (1.5, float(np.float32(0.5 * np.sqrt(2)))),
                                       (1.25, float(np.float32(0.25 * np.sqrt(5)))), (1.001, 1e-3)])
def test_compat_adversarial_threshold_ties(tr_mod, scale, tau):
    # lattice points: thousands of pairs sit exactly on (or one rounding away from) the threshold, the worst
    # case for the certified sqrt-free filter; C must still equal the oracle's float32 tree bit for bit
    g = np.stack(np.meshgrid(np.arange(9), np.arange(9), np.arange(8), indexing="ij"), -1).reshape(-1, 3)
    src = g.astype(np.float32)
    dst = (g * scale + np.array([0.25, -3.0, 7.0])).astype(np.float32)
    n = src.shape[0]
    tr = tr_mod(tau, 50, 2, 0.01, max_n=n)
    tr.register(src, dst)
    ref, e, near, _ = oracle.compat(src, dst, tau)
    assert near > 100  # the case really is adversarial
    got = tr.bits(0)
    assert (got == ref).all(), int((got != ref).sum())


@pytest.mark.parametrize("path", [0, 2])
@pytest.mark.parametrize("key,n", [("B", 2500), ("C", 3000), ("D", 1800)])
def test_heavy_block_paths_agree_with_oracle(tr_mod, path, key, n):
    # every row eligible for the dense block: tensor-core epilogue emission vs CUDA-core D + k_emit_hh
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=2, n=n)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n)
    tr.set_option("sc2_path", path)
    tr.set_option("heavy_min_rows", 1)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("key,n", [("B", 2100), ("D", 1337)])
def test_compat_variants_agree_with_oracle(tr_mod, variant, key, n):
    # compat tilings: row pairs x 2 columns (default), column pairs x 2 tiles, row pairs x 1 column
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=3, n=n)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n)
    tr.set_option("compat_variant", variant)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


def test_heavy_block_batch_mixed(tr_mod):
    # the persistent tensor-core kernel walks one (pair, tile) list across pairs with different |H|,
    # including pairs with no dense block (tiny / empty) between them
    cfg = synth.CONFIGS["B"]
    sizes = [1500, 40, 2200, 0, 900, 2600]
    srcs, dsts = [], []
    for p, n in enumerate(sizes):
        inst = synth.workload_instance(synth.CONFIGS["BCD"[p % 3]], pair=30 + p, n=max(n, 1))
        srcs.append(inst["src"][:n])
        dsts.append(inst["dst"][:n])
    n = np.array(sizes, np.int32)
    off = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=max(sizes), max_batch=len(sizes))
    tr.set_option("heavy_min_rows", 1)
    res = tr.register_batch(np.concatenate(srcs), np.concatenate(dsts), off, n)
    for p in range(len(sizes)):
        if sizes[p] >= 3:
            r = {k: res[p][k] for k in res.dtype.names}
            compare_pair(tr, p, srcs[p], dsts[p], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)


def test_heavy_block_batch_beyond_smem_table(tr_mod):
    # batches larger than the tensor-core kernel's shared-memory tile table (1024 pairs) walk the per-pair
    # state in global memory instead; every pair's result must equal the all-popcount path's, and sampled
    # pairs on both sides of pair 1024 must equal the oracle
    cfg = synth.CONFIGS["B"]
    pairs, nn = 1100, 400
    insts = [synth.workload_instance(cfg, pair=2000 + p, n=nn) for p in range(pairs)]
    src = np.concatenate([x["src"] for x in insts])
    dst = np.concatenate([x["dst"] for x in insts])
    off = np.arange(pairs, dtype=np.int64) * nn
    n = np.full(pairs, nn, np.int32)
    tc = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, max_batch=pairs)
    tc.set_option("heavy_min_rows", 1)
    pc = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, max_batch=pairs)
    pc.set_option("sc2_path", 1)
    rt = tc.register_batch(src, dst, off, n)
    rp = pc.register_batch(src, dst, off, n)
    assert rt.tobytes() == rp.tobytes()
    assert int(tc.intermediate(pairs - 1, I_STATE)["heavy_h"]) > 0  # the tensor-core block ran
    for p in (3, 1023, 1024, pairs - 1):
        r = {k: rt[p][k] for k in rt.dtype.names}
        compare_pair(tc, p, insts[p]["src"], insts[p]["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)


def test_graph_replay_matches_direct_launches(tr_mod):
    # the first call of a shape is captured into a CUDA graph, later calls replay it on new inputs; results
    # must equal a context that launches directly, for every call and across shape changes
    cfg = synth.CONFIGS["B"]
    g = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2500, max_batch=3)
    d = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2500, max_batch=3)
    d.set_option("cuda_graph", 0)
    calls = [(2000, [40]), (2000, [41]), (2500, [42, 43]), (2000, [44]), (2500, [45, 46])]
    for n, pairs in calls:
        insts = [synth.workload_instance(cfg, pair=p, n=n) for p in pairs]
        src = np.concatenate([x["src"] for x in insts])
        dst = np.concatenate([x["dst"] for x in insts])
        off = np.arange(len(pairs), dtype=np.int64) * n
        nn = np.full(len(pairs), n, np.int32)
        rg = g.register_batch(src, dst, off, nn)
        rd = d.register_batch(src, dst, off, nn)
        assert rg.tobytes() == rd.tobytes(), (n, pairs)
    assert g.launch_count == d.launch_count


def test_pipelined_host_batch_matches_single_launch(tr_mod):
    # >= 16 pairs from host memory run as 4 sub-batches (workspace views, overlapped H2D); results must be
    # identical to one launch sequence, including empty / too-small pairs at sub-batch edges
    cfg = synth.CONFIGS["D"]
    sizes = [1200, 0, 900, 1500, 2, 1100, 1300, 700, 1500, 1000, 1200, 800, 1400, 600, 1500, 1250, 0, 1000, 950]
    srcs, dsts = [], []
    for p, n in enumerate(sizes):
        inst = synth.workload_instance(cfg, pair=60 + p, n=max(n, 1))
        srcs.append(inst["src"][:n])
        dsts.append(inst["dst"][:n])
    n = np.array(sizes, np.int32)
    off = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    src, dst = np.concatenate(srcs), np.concatenate(dsts)
    a = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=1500, max_batch=len(sizes))
    b = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=1500, max_batch=len(sizes))
    b.set_option("pipeline_host_inputs", 0)
    ra = a.register_batch(src, dst, off, n)
    rb = b.register_batch(src, dst, off, n)
    assert ra.tobytes() == rb.tobytes()
    for p in (0, 5, 14):
        r = {k: ra[p][k] for k in ra.dtype.names}
        compare_pair(a, p, srcs[p], dsts[p], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)


@pytest.mark.parametrize("pairs_per_thread", [1, 2])
def test_score_packings_agree_with_oracle(tr_mod, pairs_per_thread):
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=17, n=1700)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=1700)
    tr.set_option("score_pairs", pairs_per_thread)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


def test_wide_rows_general_paths(tr_mod):
    # n = 8500: W = 268 > 256 words per row (degree pass general path, 16-word-per-lane SC2 kernels,
    # 2-row sparse groups); 3DLoMatch-shaped so the oracle's literal SC^2 loop stays within seconds
    cfg = synth.CONFIGS["C"]
    inst = synth.workload_instance(cfg, pair=1, n=8500)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=8500)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("widen", [0, 1, 40, 200])
@pytest.mark.parametrize("key", ["B", "D"])
def test_heavy_set_rules_agree_with_oracle(tr_mod, widen, key):
    # which rows the tensor-core block takes (heavy_widen: only at no extra block, every non-sparse row, or an
    # explicit degree threshold, possibly below the sparse-row list length) only moves edges between the
    # assembly paths: results are the oracle's whatever the rule
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=23, n=2400)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2400)
    tr.set_option("heavy_widen", widen)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("policy", [0, 2])
def test_tensor_core_l2_policies_agree_with_oracle(tr_mod, policy):
    # the L2 policy of the operand loads is a cache hint: same results
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=24, n=2300)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2300)
    tr.set_option("mma_l2_policy", policy)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("cap", [256, 512])
def test_heavy_cap_raises_threshold(tr_mod, cap):
    # more high-degree rows than the dense block holds: the degree threshold is raised until |H| <= cap
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=21, n=2600)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2600)
    tr.set_option("heavy_cap", cap)
    tr.set_option("heavy_min_rows", 1)
    res = tr.register(inst["src"], inst["dst"])
    from paper_2507_01439_b200._binding import I_STATE

    st = tr.intermediate(0, I_STATE)
    assert 0 < st["heavy_h"] <= cap
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("cpi", [1, 2, 64])
def test_sc2_row_split_agrees_with_oracle(tr_mod, cpi):
    # dense rows split into work items of cpi 32-word chunks (small batches) or whole rows (large batches)
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=23, n=2300)
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2300)
    tr.set_option("sc2_chunks", cpi)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)


@pytest.mark.parametrize("fp4", [0, 1])
@pytest.mark.parametrize("key,n", [("B", 2600), ("D", 2100), ("E", None)])
def test_tensor_core_formats_agree_with_oracle(tr_mod, fp4, key, n):
    # int8 operands (kind::i8) vs packed e2m1 operands with unit block scales (kind::mxf4.block_scale)
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=29, n=n)
    nn = inst["src"].shape[0]
    tr = tr_mod(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn)
    tr.set_option("mma_fp4", fp4)
    tr.set_option("heavy_min_rows", 1)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)
