"""graph_mode = 1 (undirected SC^2 graph, Table 5 row 10; reading r9) vs the oracle, through the C ABI.
Needs a B200: `pytest -m gpu`."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_compare import compare_pair
from tests.helpers import py_triangles

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def TR():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import TurboReg

    return TurboReg


@pytest.mark.parametrize("key,n", [("A", None), ("B", 2000), ("C", 1500), ("D", 1700)])
def test_sc2_mode_parity(TR, key, n):
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=7, n=n)
    nn = inst["src"].shape[0]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, graph_mode=1, max_n=nn)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res,
                 graph_mode=1)


@pytest.mark.parametrize("k1,k2", [(1, 1), (5, 3), (40, 8), (300, 9)])
def test_sc2_mode_budgets(TR, k1, k2):
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=4)
    tr = TR(cfg.tau, k1, k2, cfg.inlier_threshold, graph_mode=1, max_n=cfg.n)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, k1, k2, cfg.inlier_threshold, result=res, graph_mode=1)


@pytest.mark.parametrize("density", [0.1, 0.3])
def test_sc2_mode_full_budget_every_triangle_once(TR, density):
    # App. C: with K1 = all edges and K2 = N the SC^2-mode search finds every triangle three times (once
    # per edge as pivot); after de-duplication each appears exactly once, in canonical order
    n = 30  # K1 * K2 = 435 * 28 stays within the canonical-sort capacity
    C = synth.erdos_renyi(n, density, 77)
    tr = TR(0.01, n * (n - 1) // 2, n - 2, 0.1, graph_mode=1, max_n=n)
    tr.pgs_from_adjacency(C)
    from paper_2507_01439_b200._binding import I_CLIQUES

    cl = tr.intermediate(0, I_CLIQUES)
    cl = cl[cl[:, 0] >= 0]
    assert sorted(map(tuple, cl[:, :3].tolist())) == sorted(py_triangles(C))
    G = oracle.sc2(C)
    raw, _ = oracle.pgs(G, oracle.select_pivots(G, n * n), n - 2)
    assert len(raw) == 3 * len(cl)
    ref = oracle.canonical(raw, dedup=True)
    assert (cl == ref).all()  # same list, same canonical order


def test_sc2_mode_budget_limit_rejected(TR):
    with pytest.raises(Exception):
        TR(0.01, 10000, 2, 0.1, graph_mode=1, max_n=100)


@pytest.mark.parametrize("key", ["B", "C", "D"])
def test_sc2_mode_parity_baseline_size(TR, key):
    """graph_mode = 1 at the BASELINE size (N = 5000, the config's own K1, K2): every intermediate and the
    winner against the oracle (SC^2 mode had been parity-tested only up to N = 2000)."""
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=17)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, graph_mode=1, max_n=cfg.n)
    res = tr.register(inst["src"], inst["dst"])
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res,
                 graph_mode=1)
