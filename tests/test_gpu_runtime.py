"""Runtime contracts of the C ABI on the GPU: edge capacity and its overflow status, workspace size,
asynchronous calls on different streams, set_params / set_option reallocation (the reading-r22 workflow
τ = 0.25·pr), deterministic MAE/MSE sums, point_resolution beyond max_n, STAGE_TIMING.
Every registration is compared with the oracle.  Needs a B200: `pytest -m gpu`."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_compare import compare_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def TR():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import TurboReg

    return TurboReg


def _batch(insts):
    n = np.array([i["src"].shape[0] for i in insts], np.int32)
    off = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    return np.concatenate([i["src"] for i in insts]), np.concatenate([i["dst"] for i in insts]), off, n


def test_edge_capacity_overflow_is_per_pair(TR):
    """A pair whose graph has more edges than the create-time capacity reports EDGE_CAPACITY (8) with its true
    edge count; the other pairs of the batch are unaffected and match the oracle."""
    cfg = synth.CONFIGS["A"]
    big = synth.workload_instance(cfg, pair=3)
    small = synth.workload_instance(cfg, pair=4, n=260)
    e_big = oracle.estimate(big["src"], big["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)["num_edges"]
    e_small = oracle.estimate(small["src"], small["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)["num_edges"]
    assert e_small < e_big
    cap = (e_small + e_big) // 2 // 4 * 4
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=3, max_edges=cap)
    src, dst, off, n = _batch([small, big, small])
    res = tr.register_batch(src, dst, off, n)
    assert [int(s) for s in res["status"]] == [0, 8, 0]
    assert int(res[1]["num_edges"]) == e_big
    assert np.all(res[1]["R"] == 0) and int(res[1]["num_pivots"]) == 0
    for p in (0, 2):
        r = {k: res[p][k] for k in res.dtype.names}
        compare_pair(tr, p, small["src"], small["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)
    # exactly at capacity: no overflow
    tr2 = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=1, max_edges=e_big)
    r = tr2.register(big["src"], big["dst"])
    compare_pair(tr2, 0, big["src"], big["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)


def test_workspace_per_pair_at_bench_density(TR):
    """N = 5000 with the bench's density bound (1/8 of all pairs, 3x config E's measured 4.35 %): at most
    20 MB of workspace per pair, so the 1623-pair sweep fits one GPU in about 31 GB."""
    cfg = synth.CONFIGS["E"]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=8, max_density=0.125)
    per_pair = tr.workspace_bytes / 8
    assert per_pair <= 20e6, per_pair
    full = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=8)
    assert full.workspace_bytes > tr.workspace_bytes + 8 * 4 * (cfg.n * (cfg.n - 1) // 2 - 1562500) * 0.99


def test_async_calls_on_two_streams(TR):
    """Back-to-back asynchronous calls (device inputs and outputs) with different batch sizes and n on two
    streams: each call sees its own descriptors and waits for the previous call's workspace use."""
    import torch

    from paper_2507_01439_b200 import RESULT_DTYPE

    cfg = synth.CONFIGS["A"]
    ia = [synth.workload_instance(cfg, pair=40 + k) for k in range(3)]
    ib = [synth.workload_instance(cfg, pair=50, n=420)]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=3)
    sa, da, oa, na = _batch(ia)
    sb, db, ob, nb = _batch(ib)
    ref_a = tr.register_batch(sa, da, oa, na)
    ref_b = tr.register_batch(sb, db, ob, nb)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    dsa, dda = torch.from_numpy(sa).cuda(), torch.from_numpy(da).cuda()
    dsb, ddb = torch.from_numpy(sb).cuda(), torch.from_numpy(db).cuda()
    torch.cuda.synchronize()
    outs = []
    for rep in range(4):
        o1 = torch.zeros(3 * 104, dtype=torch.uint8, device="cuda")
        o2 = torch.zeros(104, dtype=torch.uint8, device="cuda")
        o1.record_stream(s1)
        o2.record_stream(s2)
        tr.register_batch(dsa, dda, oa, na, out=o1, stream=s1.cuda_stream)
        tr.register_batch(dsb, ddb, ob, nb, out=o2, stream=s2.cuda_stream)
        outs.append((o1, o2))
    torch.cuda.synchronize()
    for o1, o2 in outs:
        assert o1.cpu().numpy().view(RESULT_DTYPE).tobytes() == ref_a.tobytes()
        assert o2.cpu().numpy().view(RESULT_DTYPE).tobytes() == ref_b.tobytes()


def test_set_params_tau_from_resolution_round_trip(TR):
    """Reading r22 workflow: pr = point_resolution(source cloud) → τ = 0.25·pr → set_params →
    register, against the oracle at that τ; then K1, K2 and graph_mode changed on the live context."""
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=7, n=2500)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=2500, max_batch=1)
    r0 = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r0)
    pr = tr.point_resolution(inst["src"])
    assert pr == oracle.point_resolution(inst["src"])
    tau = float(np.float32(0.25 * pr))
    tr.set_params(tau=tau)
    r1 = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r1)
    for k1, k2, gm in ((300, 3, 0), (1500, 2, 1), (1000, 2, 0)):
        tr.set_params(tau=cfg.tau, k1=k1, k2=k2, graph_mode=gm)
        r = tr.register(inst["src"], inst["dst"])
        compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, k1, k2, cfg.inlier_threshold, result=r,
                     graph_mode=gm)
    with pytest.raises(Exception):
        tr.set_params(k1=0)
    # a rejected set_params leaves the context usable with its previous parameters
    assert tr.params.k1 == 1000
    r = tr.register(inst["src"], inst["dst"])
    assert r["status"] == 0 and tuple(r["clique"]) == tuple(r0["clique"])


def test_set_option_relayout_keeps_results(TR):
    """mma_fp4 = 0 (uint8 X, kind::i8) and sc2_path = 2 (CUDA-core D) reallocate the operand block; results
    stay identical to the default packed-e2m1 layout."""
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=8)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=1)
    base = tr.register(inst["src"], inst["dst"])
    ws0 = tr.workspace_bytes
    from paper_2507_01439_b200._binding import I_EDGES, I_STATE

    e0 = tr.intermediate(0, I_EDGES)[1].copy()
    assert tr.intermediate(0, I_STATE)["heavy_h"] > 0
    for opt, val in (("mma_fp4", 0), ("sc2_path", 2), ("sc2_path", 0), ("mma_fp4", 1)):
        tr.set_option(opt, val)
        r = tr.register(inst["src"], inst["dst"])
        assert {k: r[k] for k in ("clique", "inlier_count", "num_edges")} == \
            {k: base[k] for k in ("clique", "inlier_count", "num_edges")}
        assert (tr.intermediate(0, I_EDGES)[1] == e0).all()
    assert tr.workspace_bytes == ws0


def test_hyp_errors_deterministic(TR):
    """MAE/MSE partial sums go to fixed per-segment slots added in order: identical bits on every run."""
    from paper_2507_01439_b200._binding import I_ERRORS

    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=12)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, hyp_errors=True)
    tr.register(inst["src"], inst["dst"])
    e0 = tr.intermediate(0, I_ERRORS).copy()
    for _ in range(3):
        tr.register(inst["src"], inst["dst"])
        assert tr.intermediate(0, I_ERRORS).tobytes() == e0.tobytes()


def test_point_resolution_beyond_max_n(TR):
    cfg = synth.CONFIGS["A"]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=500, max_batch=1)
    cloud = np.random.default_rng(5).uniform(-1, 1, size=(6000, 3)).astype(np.float32)
    assert tr.point_resolution(cloud) == oracle.point_resolution(cloud)
    inst = synth.workload_instance(cfg, pair=2)
    r = tr.register(inst["src"], inst["dst"])  # the context is unaffected
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=r)


def test_stage_timing_fills_stage_ms(TR):
    """TURBOREG_F_STAGE_TIMING: stage_ms = (graph, PGS, model) in App. F.3's naming, all positive,
    summing to no more than the call's wall time; results unchanged."""
    import time

    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=13)
    plain = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n)
    timed = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, stage_timing=True)
    a = plain.register(inst["src"], inst["dst"])
    timed.register(inst["src"], inst["dst"])
    t0 = time.perf_counter()
    b = timed.register(inst["src"], inst["dst"])
    wall_ms = 1e3 * (time.perf_counter() - t0)
    st = b["stage_ms"]
    assert all(x > 0 for x in st), st
    assert sum(st) <= wall_ms, (st, wall_ms)
    assert tuple(a["clique"]) == tuple(b["clique"]) and a["inlier_count"] == b["inlier_count"]
    assert tuple(a["stage_ms"]) == (0.0, 0.0, 0.0)


def test_independent_contexts_concurrently(TR):
    """Independent contexts may run concurrently: two threads, each with its own context."""
    import threading

    cfg = synth.CONFIGS["A"]
    insts = [synth.workload_instance(cfg, pair=60 + k) for k in range(2)]
    refs = [oracle.estimate(i["src"], i["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold) for i in insts]
    out = [None, None]

    def work(k):
        tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n)
        rs = [tr.register(insts[k]["src"], insts[k]["dst"]) for _ in range(5)]
        out[k] = rs
        tr.close()

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(2):
        for r in out[k]:
            assert r["status"] == refs[k]["status"] == 0
            assert tuple(r["clique"]) == tuple(refs[k]["clique"]) and r["inlier_count"] == refs[k]["inlier_count"]


def test_create_destroy_releases_device_memory(TR):
    """Every context owns one workspace allocation plus its streams, events, graphs and pinned slots; destroying
    it returns them: 40 create / register (graph captured) / set_option re-layout / destroy cycles leave the
    device's free memory where it was (within 64 MiB of allocator slack)."""
    import torch

    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=3, n=1200)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for k in range(40):
        tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=1200, max_batch=4)
        for _ in range(2):  # the second call replays the captured graph
            assert tr.register(inst["src"], inst["dst"])["status"] == 0
        if k % 4 == 0:
            tr.set_option("mma_fp4", 0)  # workspace re-layout (allocate new, free old)
            assert tr.register(inst["src"], inst["dst"])["status"] == 0
        tr.close()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, (free0, free1)


def test_binding_rejects_bad_extents(TR):
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=1)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=2)
    with pytest.raises(ValueError):
        tr.register_batch(inst["src"], inst["dst"], [0, 100], [500, 500])  # past the rows
    with pytest.raises(ValueError):
        tr.register(inst["src"], inst["dst"][:-1])
    with pytest.raises(ValueError):
        tr.register(inst["src"][:, :2], inst["dst"][:, :2])
    import torch

    with pytest.raises(ValueError):
        tr.register_batch(torch.from_numpy(inst["src"]).cuda(), torch.from_numpy(inst["dst"]).cuda(), [0], [500],
                          out=torch.zeros(50, dtype=torch.uint8, device="cuda"))


@pytest.mark.parametrize("key,n", [("A", None), ("B", 5000), ("D", 2000)])
def test_row_sums_equal_twice_triangle_counts(TR, key, n):
    """r_i = Σ_j Ĝ_ij (north star: "per-row SC² sums"): equal to the oracle's Ĝ row sums, and to 2·t_i with
    t_i the triangles through i (App. B), computed here as diag(C³)/2 with numpy on the GPU's own C
    (a library matmul, independent of oracle/)."""
    from paper_2507_01439_b200._binding import I_ROWSUM

    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=21, n=n)
    nn = inst["src"].shape[0]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, row_sums=True)
    r = tr.register(inst["src"], inst["dst"])
    rs = tr.intermediate(0, I_ROWSUM)
    ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, trace=True)
    assert (rs == ref["G"].sum(axis=1)).all()
    C = tr.bits(0).astype(np.float64)
    two_t = np.einsum("ij,ji->i", C @ C, C)  # diag(C^3) = 2 t_i
    assert (rs == two_t.astype(np.int64)).all()
    plain = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn)
    assert plain.register(inst["src"], inst["dst"])["clique"] == r["clique"]
    with pytest.raises(Exception):
        plain.intermediate(0, I_ROWSUM)


def _oracle_ranking(ref, metric):
    ok = ref["hyp_degenerate"] == 0
    cl = ref["cliques"][ok]
    cnt = ref["hyp_count"][ok].astype(np.int64)
    err = {"in": -cnt, "mae": ref["hyp_mae"][ok], "mse": ref["hyp_mse"][ok]}[metric]
    order = np.lexsort((cl[:, 2], cl[:, 1], cl[:, 0], -cl[:, 3], err))
    return cl[order], err[order]


@pytest.mark.parametrize("metric", ["in", "mae", "mse"])
@pytest.mark.parametrize("key,n,graph_mode", [("A", None, 0), ("B", 5000, 0), ("C", 3000, 1)])
def test_ranked_hypotheses_match_oracle(TR, metric, key, n, graph_mode):
    """Ranked hypothesis list (App. F.1): the oracle's per-hypothesis IN / MAE / MSE
    sorted by (metric, S desc, (i,j,z) asc); entry 0 under the context's own metric is the returned T*."""
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=23, n=n)
    nn = inst["src"].shape[0]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, hyp_errors=True, graph_mode=graph_mode,
            rank_metric=metric)
    res = tr.register(inst["src"], inst["dst"])
    got = tr.ranked_hypotheses(0, metric)
    ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, trace=True,
                          graph_mode=graph_mode)
    want_cl, want_key = _oracle_ranking(ref, metric)
    assert len(got) == len(want_cl) == res["hypotheses_evaluated"]
    gcl = np.concatenate([got["clique"], got["clique_weight"][:, None]], axis=1)
    if metric == "in":
        assert (gcl == want_cl).all()
        assert (got["inlier_count"] == -want_key).all()
    else:  # float64 sums in another order: equal within 1e-12, so only near-equal keys may swap
        gkey = got[metric]
        assert np.all(np.abs(np.sort(gkey) - np.sort(want_key)) <= 1e-12 * np.abs(want_key))
        assert np.all(np.diff(gkey) >= 0)
        same = np.all(gcl == want_cl, axis=1)
        for k in np.nonzero(~same)[0]:  # a swap is only allowed among keys equal to 1e-12
            assert abs(gkey[k] - want_key[k]) <= 1e-12 * abs(want_key[k])
    assert tuple(got[0]["clique"]) == tuple(res["clique"])
    top = tr.ranked_hypotheses(0, metric, top_k=5)
    assert top.tobytes() == got[:5].tobytes()


def test_api_argument_errors(TR):
    """Argument failures return INVALID_ARGUMENT (raised by the binding) and leave the context usable."""
    import ctypes

    from paper_2507_01439_b200._binding import Params, Status, TurboRegError, library

    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=3)
    lib = library()
    h = ctypes.c_void_p()
    prm = Params(cfg.tau, 0.0, cfg.k1, cfg.k2, cfg.inlier_threshold, 0, 0)
    assert lib.turboreg_create_ex(ctypes.byref(prm), 0, 500, 1, -1, ctypes.byref(h)) == Status.INVALID_ARGUMENT
    assert lib.turboreg_create_ex(ctypes.byref(prm), 0, 2, 1, 0, ctypes.byref(h)) == Status.INVALID_ARGUMENT
    bad = Params(cfg.tau, 0.0, cfg.k1, cfg.k2, cfg.inlier_threshold, 0, 0x40)  # unknown flag
    assert lib.turboreg_create_ex(ctypes.byref(bad), 0, 500, 1, 0, ctypes.byref(h)) == Status.INVALID_ARGUMENT
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n)
    with pytest.raises(TurboRegError):
        tr.set_option("no_such_option", 1)
    with pytest.raises(TurboRegError):
        tr.set_option("heavy_cap", 100)  # not a multiple of 256
    with pytest.raises(TurboRegError):
        tr.ranked_hypotheses(0, "in")  # no call yet
    r = tr.register(inst["src"], inst["dst"])
    with pytest.raises(TurboRegError):
        tr.ranked_hypotheses(0, "mae")  # errors not accumulated by this context
    with pytest.raises(TurboRegError):
        tr.ranked_hypotheses(1, "in")  # no such pair in the last call
    with pytest.raises(TurboRegError):
        tr.split_begin(inst["src"], inst["dst"], 2, 2)  # rank outside [0, world)
    assert tr.split_begin(inst["src"][:2], inst["dst"][:2], 0, 2) == 2  # too few points: the pair's status
    r2 = tr.register(inst["src"], inst["dst"])
    assert tuple(r2["clique"]) == tuple(r["clique"]) and r2["inlier_count"] == r["inlier_count"]
    assert len(tr.ranked_hypotheses(0, "in", top_k=3)) == 3
