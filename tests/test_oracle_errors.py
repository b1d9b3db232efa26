"""Oracle MAE / MSE per hypothesis and metric-ranked selection (App. F.1, reading r20), pinned
against closed forms and an independent numpy evaluation."""
import numpy as np

import oracle
import synth


def test_unit_displacement_closed_form():
    # identity (R = I, t = 0) on y = x + (1, 0, 0): every residual is exactly (-1, 0, 0) in float32
    rng = np.random.default_rng(3)
    x = rng.uniform(-2, 2, (257, 3)).astype(np.float32)
    y = x.copy()
    y[:, 0] = (x[:, 0].astype(np.float64) + 1.0).astype(np.float32)
    exact = (y[:, 0].astype(np.float64) - x[:, 0]) == 1.0  # rows where the shift is exact in float32
    mae, mse = oracle.hypothesis_errors(x[exact], y[exact], np.eye(3), np.zeros(3))
    assert mae == 1.0 and mse == 1.0


def test_errors_match_numpy_float64():
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=2)
    R = np.asarray(inst["R"], np.float32)
    t = np.asarray(inst["t"], np.float32)
    mae, mse = oracle.hypothesis_errors(inst["src"], inst["dst"], R, t)
    r = inst["src"].astype(np.float64) @ R.astype(np.float64).T + t.astype(np.float64) - inst["dst"].astype(np.float64)
    d2 = (r * r).sum(1)
    assert abs(mae - np.sqrt(d2).mean()) <= 1e-5 * np.sqrt(d2).mean()
    assert abs(mse - d2.mean()) <= 1e-5 * d2.mean()


def test_rank_metric_selects_minimum_error():
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=5)
    for metric, key in ((1, "hyp_mae"), (2, "hyp_mse")):
        ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, trace=True,
                              rank_metric=metric)
        ok = ref["hyp_degenerate"] == 0
        errs = ref[key][ok]
        assert ref["status"] == 0
        assert (ref["mae"] if metric == 1 else ref["mse"]) == errs.min()
        c = ref["cliques"][ok][np.argmin(errs)]  # first minimum in canonical order
        assert tuple(c[:3]) == tuple(ref["clique"])
        # independent check of every listed error against numpy float64
        for k in np.nonzero(ok)[0][:25]:
            R, t = ref["hyp_R"][k].astype(np.float64), ref["hyp_t"][k].astype(np.float64)
            d2 = ((inst["src"].astype(np.float64) @ R.T + t - inst["dst"]) ** 2).sum(1)
            want = np.sqrt(d2).mean() if metric == 1 else d2.mean()
            assert abs(ref[key][k] - want) <= 1e-5 * want
    # inlier-number selection is unchanged by the extra outputs
    a = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)
    assert a["status"] == 0 and a["inlier_count"] > 0
