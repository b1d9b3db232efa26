"""MAE / MSE per hypothesis and metric-ranked selection (App. F.1, reading r20) vs the oracle,
through the C ABI.  Needs a B200: `pytest -m gpu`."""
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


def _errors_by_clique(tr, pair):
    from paper_2507_01439_b200._binding import I_CLIQUES, I_ERRORS

    cl = tr.intermediate(pair, I_CLIQUES)
    er = tr.intermediate(pair, I_ERRORS)
    return {tuple(c[:3]): e for c, e in zip(cl.tolist(), er) if c[0] >= 0}


@pytest.mark.parametrize("key,n", [("A", None), ("B", 1500), ("D", 1200)])
def test_hypothesis_errors_match_oracle(TR, key, n):
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=9, n=n)
    nn = inst["src"].shape[0]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, hyp_errors=True)
    res = tr.register(inst["src"], inst["dst"])
    # the inlier-number path is untouched by the extra accumulation
    compare_pair(tr, 0, inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, result=res)
    ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, trace=True)
    got = _errors_by_clique(tr, 0)
    ok = ref["hyp_degenerate"] == 0
    for c, mae, mse in zip(ref["cliques"][ok], ref["hyp_mae"][ok], ref["hyp_mse"][ok]):
        g = got[tuple(c[:3])]
        assert abs(g[0] - mae) <= 1e-12 * mae and abs(g[1] - mse) <= 1e-12 * mse


@pytest.mark.parametrize("metric", ["mae", "mse"])
@pytest.mark.parametrize("key,n,graph_mode", [("A", None, 0), ("B", 1500, 0), ("C", 1500, 1)])
def test_rank_by_error_selects_oracle_winner(TR, metric, key, n, graph_mode):
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=11, n=n)
    nn = inst["src"].shape[0]
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, rank_metric=metric, graph_mode=graph_mode)
    res = tr.register(inst["src"], inst["dst"])
    ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold,
                          graph_mode=graph_mode, rank_metric=1 if metric == "mae" else 2)
    assert res["status"] == ref["status"] == 0
    assert tuple(res["clique"]) == tuple(ref["clique"])
    assert res["inlier_count"] == ref["inlier_count"]
    got = _errors_by_clique(tr, 0)[tuple(res["clique"])]
    want = ref["mae"] if metric == "mae" else ref["mse"]
    assert abs(got[0 if metric == "mae" else 1] - want) <= 1e-12 * want


@pytest.mark.parametrize("key", ["B", "D"])
def test_hypothesis_errors_baseline_size(TR, key):
    """MAE / MSE of every hypothesis at N = 5000 (the BASELINE size) within 1e-12 relative of the oracle's
    sequential float64 sums, and both error rankings select the oracle's winner."""
    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=19)
    ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, trace=True)
    tr = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, hyp_errors=True)
    res = tr.register(inst["src"], inst["dst"])
    assert res["status"] == ref["status"] == 0 and tuple(res["clique"]) == tuple(ref["clique"])
    got = _errors_by_clique(tr, 0)
    ok = ref["hyp_degenerate"] == 0
    for c, mae, mse in zip(ref["cliques"][ok], ref["hyp_mae"][ok], ref["hyp_mse"][ok]):
        g = got[tuple(c[:3])]
        assert abs(g[0] - mae) <= 1e-12 * mae and abs(g[1] - mse) <= 1e-12 * mse
    for metric, rm in (("mae", 1), ("mse", 2)):
        t2 = TR(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, rank_metric=metric)
        r2 = t2.register(inst["src"], inst["dst"])
        ref2 = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, rank_metric=rm)
        assert tuple(r2["clique"]) == tuple(ref2["clique"]) and r2["inlier_count"] == ref2["inlier_count"]
