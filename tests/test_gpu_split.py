"""NEXT(1): one pair split over G ranks (include/turboreg.h "NEXT(1)", paper_2507_01439_b200/split.py), run as
G logical ranks on one GPU (emulate_split: the same phases and buffers, exchanges as sums).  Results must be
bit-identical to the single-rank path and equal to the oracle (n = 8500), and at n = 32768 identical to the
single-rank path with sampled rows of C checked against Eq. 1's float32 tree in numpy.
Needs a B200: `pytest -m gpu`."""
import numpy as np
import pytest

import oracle
import synth
from paper_2507_01439_b200._binding import I_BITS, I_EDGES, I_PIVOTS, I_STATE

pytestmark = pytest.mark.gpu

KEYS = ("status", "inlier_count", "clique", "clique_weight", "num_pivots", "num_cliques", "hypotheses_evaluated",
        "num_edges")


@pytest.fixture(scope="module")
def TR():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import TurboReg

    return TurboReg


def _same(a, b):
    for k in KEYS:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (k, a[k], b[k])
    assert np.asarray(a["R"]).tobytes() == np.asarray(b["R"]).tobytes()
    assert np.asarray(a["t"]).tobytes() == np.asarray(b["t"]).tobytes()


def _run(TR, cfg, inst, G, max_n, **kw):
    from paper_2507_01439_b200.split import emulate_split

    engines = [TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=max_n, **kw) for _ in range(G)]
    res = emulate_split(engines, inst["src"], inst["dst"])
    return res, engines


@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_split_equals_single_rank_and_oracle(TR, G):
    cfg = synth.CONFIGS["B"]
    inst = synth.workload_instance(cfg, pair=31, n=8500)
    one = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=8500)
    ref1 = one.register(inst["src"], inst["dst"])
    res, engines = _run(TR, cfg, inst, G, 8500)
    _same(res, ref1)
    # after the exchanges every rank holds the whole graph and edge list
    for e in engines:
        assert (e.intermediate(0, I_BITS) == one.intermediate(0, I_BITS)).all()
        r1, w1 = one.intermediate(0, I_EDGES)
        r2, w2 = e.intermediate(0, I_EDGES)
        assert (r1 == r2).all() and (w1 == w2).all()
        assert (e.intermediate(0, I_PIVOTS) == one.intermediate(0, I_PIVOTS)).all()
    if G == 2:
        ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)
        for k in ("status", "inlier_count", "clique_weight", "num_pivots", "num_cliques", "hypotheses_evaluated",
                  "num_edges"):
            assert res[k] == ref[k], (k, res[k], ref[k])
        assert tuple(res["clique"]) == tuple(ref["clique"])
        assert np.abs(np.asarray(res["t"], np.float64) - ref["t"]).max() <= 1e-5


def _eq1_rows(src, dst, rows, tau):
    """Rows of C by Eq. 1 in numpy float32 (reading r1's tree, every op correctly rounded, no FMA)."""
    s = src.astype(np.float32)
    d = dst.astype(np.float32)
    out = []
    for i in rows:
        dx, dy, dz = (s[i, 0] - s[:, 0]), (s[i, 1] - s[:, 1]), (s[i, 2] - s[:, 2])
        a = np.sqrt((dx * dx + dy * dy) + dz * dz)
        ex, ey, ez = (d[i, 0] - d[:, 0]), (d[i, 1] - d[:, 1]), (d[i, 2] - d[:, 2])
        b = np.sqrt((ex * ex + ey * ey) + ez * ez)
        c = np.abs(a - b) <= np.float32(tau)
        c[i] = False
        out.append(c)
    return np.array(out)


@pytest.mark.parametrize("G", [2, 4])
def test_split_large_n(TR, G):
    cfg = synth.CONFIGS["B"]
    n = 32768
    inst = synth.workload_instance(cfg, pair=33, n=n)
    one = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n, max_density=0.1)
    ref1 = one.register(inst["src"], inst["dst"])
    res, engines = _run(TR, cfg, inst, G, n, max_density=0.1)
    _same(res, ref1)
    assert res["status"] == 0 and synth.rotation_error_deg(np.asarray(res["R"]).reshape(3, 3), inst["R"]) <= 2
    st = engines[-1].intermediate(0, I_STATE)
    W = st["W"]
    rows = np.random.default_rng(G).choice(n, 24, replace=False)
    words = engines[-1].intermediate(0, I_BITS).reshape(n, W)[rows]
    got = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :n].astype(bool)
    assert (got == _eq1_rows(inst["src"], inst["dst"], rows, cfg.tau)).all()


def test_split_statuses(TR):
    from paper_2507_01439_b200.split import emulate_split

    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=2)
    engines = [TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n) for _ in range(2)]
    assert emulate_split(engines, inst["src"][:2], inst["dst"][:2])["status"] == 2
    one = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n)
    _same(emulate_split(engines, inst["src"], inst["dst"]), one.register(inst["src"], inst["dst"]))
    # the split covers the paper's O2 path only
    sc2 = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, graph_mode=1)
    with pytest.raises(Exception):
        sc2.split_begin(inst["src"], inst["dst"], 0, 2)
