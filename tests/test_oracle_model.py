"""Pins for oracle steps 7-9 (Kabsch, inlier count, argmax) and the end-to-end oracle: exact recovery of
planted transforms (App. A.3), numpy.linalg.svd Kabsch (a library routine), closed-form
count cases, an independent float64 numpy residual count, planted-recovery success rates
(SPEC acceptance 5), and a brute-force argmax over every triangle on tiny inputs."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import numpy_kabsch, py_triangles, random_rotation, rot_angle_deg


@pytest.mark.parametrize("m", [3, 4, 7, 50])
def test_kabsch_exact_recovery(m):
    rng = np.random.default_rng(m)
    for _ in range(50):
        R = random_rotation(rng)
        t = rng.uniform(-2, 2, 3)
        P = rng.uniform(-1, 1, (m, 3))
        Q = P @ R.T + t
        Re, te = oracle.kabsch(P, Q)
        assert rot_angle_deg(Re, R) < 1e-6
        assert np.linalg.norm(te - t) < 1e-9
        assert abs(np.linalg.det(Re) - 1) < 1e-9 and np.abs(Re.T @ Re - np.eye(3)).max() < 1e-9


def test_kabsch_matches_numpy_svd_on_noisy_points():
    rng = np.random.default_rng(3)
    for m in (3, 3, 3, 5, 9):
        for _ in range(40):
            P = rng.uniform(-1, 1, (m, 3))
            Q = P @ random_rotation(rng).T + rng.normal(0, 0.05, (m, 3)) + 1.0
            Re, te = oracle.kabsch(P, Q)
            Rn, tn = numpy_kabsch(P, Q)
            assert np.abs(Re - Rn).max() < 1e-10 and np.abs(te - tn).max() < 1e-10


def test_kabsch_identity_and_degenerate():
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.5]], np.float64)
    R, t = oracle.kabsch(P, P)
    assert np.abs(R - np.eye(3)).max() < 1e-12 and np.abs(t).max() < 1e-12
    L = np.array([[0, 0, 0], [1, 1, 1], [2, 2, 2]], np.float64)
    assert oracle.kabsch(L, L) is None  # S:302 collinear → degenerate
    assert oracle.triangle_degenerate(*L.astype(np.float32))
    assert not oracle.triangle_degenerate(*P.astype(np.float32))


def test_kabsch_local_optimality():
    # the LS residual is ≤ that of random perturbations
    rng = np.random.default_rng(8)
    P = rng.uniform(-1, 1, (6, 3))
    Q = P @ random_rotation(rng).T + rng.normal(0, 0.03, (6, 3))
    R, t = oracle.kabsch(P, Q)
    base = ((P @ R.T + t - Q) ** 2).sum()
    for _ in range(100):
        w = rng.normal(0, 1e-3, 3)
        K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
        Rp = R @ (np.eye(3) + K + K @ K / 2)
        u, _, vt = np.linalg.svd(Rp)
        Rp = u @ vt
        assert ((P @ Rp.T + t + rng.normal(0, 1e-4, 3) - Q) ** 2).sum() >= base - 1e-12


def test_count_inliers_closed_cases():
    inst = synth.generate(200, 1.0, (1, 1, 1), 0.0, seed=2)
    R32, t32 = inst["R"].astype(np.float32), inst["t"].astype(np.float32)
    assert oracle.count_inliers(inst["src"], inst["dst"], R32, t32, 1e-3) == 200
    src = inst["src"]
    dst = src + np.array([1.0, 0, 0], np.float32)
    assert oracle.count_inliers(src, dst, np.eye(3), np.zeros(3), 0.1) == 0


def test_count_inliers_matches_float64_outside_band():
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, n=2000)
    R32, t32 = inst["R"].astype(np.float32), inst["t"].astype(np.float32)
    thr = np.float32(cfg.inlier_threshold)
    res = np.linalg.norm(inst["src"].astype(np.float64) @ R32.astype(np.float64).T + t32 - inst["dst"], axis=1)
    ref = int((res <= thr).sum())
    near = int((np.abs(res - thr) <= 1e-6 + 4 * np.spacing(thr)).sum())
    got = oracle.count_inliers(inst["src"], inst["dst"], R32, t32, thr)
    assert abs(got - ref) <= near
    # planted labels: every inlier within 6σ is counted at thr = 6σ + margin
    cnt = oracle.count_inliers(inst["src"], inst["dst"], R32, t32, 6.5 * cfg.sigma)
    assert cnt >= int(inst["inlier_mask"].sum())


def test_estimate_input_validation_and_budget():
    r = oracle.estimate(np.zeros((2, 3)), np.zeros((2, 3)), 0.01, 10, 2, 0.1)
    assert r["status"] == 2
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg)
    r = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)
    assert r["hypotheses_evaluated"] <= cfg.k1 * cfg.k2 and r["num_cliques"] <= cfg.k1 * cfg.k2
    assert r["neighbor_checks"] == r["num_pivots"] * (cfg.n - 2)


def test_estimate_exact_inliers_spec_example():
    # 100 exact inliers, τ = 1 cm, K1 = 100, K2 = 2 → exact recovery (float32 output ⇒ f32 tolerance)
    inst = synth.generate(100, 1.0, (1, 1, 1), 0.0, seed=21)
    r = oracle.estimate(inst["src"], inst["dst"], 0.01, 100, 2, 0.01)
    assert r["status"] == 0 and r["inlier_count"] == 100
    assert synth.rotation_error_deg(r["R"], inst["R"]) < 1e-3
    assert synth.translation_error(r["t"], inst["t"]) < 1e-5


def test_estimate_planted_recovery_rate():
    # SPEC acceptance 5 at config A's shape (N=500, 90% outliers): success RE ≤ 2°, TE ≤ 3 cm
    cfg = synth.CONFIGS["A"]
    ok = 0
    seeds = range(5000, 5020)
    for s in seeds:
        inst = synth.generate(cfg.n, cfg.inlier_ratio, cfg.extent, cfg.sigma, s)
        r = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)
        ok += r["status"] == 0 and synth.rotation_error_deg(r["R"], inst["R"]) <= 2 and synth.translation_error(r["t"], inst["t"]) <= 0.03
    assert ok >= 19


def test_estimate_full_budget_equals_bruteforce_argmax():
    # With K1 = all edges and K2 = N, PGS on O2 enumerates every triangle (App. C), so the winner must be
    # the best hypothesis over ALL triangles under the same key (count↓, S↓, ijz↑).
    inst = synth.generate(40, 0.4, (1, 1, 1), 0.004, seed=77)
    tau, thr = 0.015, 0.02
    r = oracle.estimate(inst["src"], inst["dst"], tau, 40 * 40, 40, thr, trace=True)
    C = r["C"]
    G = oracle.sc2(C)
    best = None
    for (i, j, z) in py_triangles(C):
        s = G[i, j] + G[i, z] + G[j, z]
        if oracle.triangle_degenerate(inst["src"][i], inst["src"][j], inst["src"][z]) or oracle.triangle_degenerate(
            inst["dst"][i], inst["dst"][j], inst["dst"][z]
        ):
            continue
        fit = oracle.kabsch(inst["src"][[i, j, z]], inst["dst"][[i, j, z]])
        if fit is None:
            continue
        cnt = oracle.count_inliers(inst["src"], inst["dst"], fit[0].astype(np.float32), fit[1].astype(np.float32), thr)
        key = (-cnt, -s, (i, j, z))
        if best is None or key < best[0]:
            best = (key, (i, j, z), cnt)
    assert best is not None
    assert r["clique"] == best[1] and r["inlier_count"] == best[2]
    assert r["num_cliques"] == len(py_triangles(C))


def test_generator_determinism_and_counts():
    a = synth.generate(1000, 0.1, (1, 1, 1), 0.005, 42)
    b = synth.generate(1000, 0.1, (1, 1, 1), 0.005, 42)
    assert (a["src"] == b["src"]).all() and (a["dst"] == b["dst"]).all()
    assert a["inlier_mask"].sum() == 100
    res = np.linalg.norm(a["src"].astype(np.float64) @ a["R"].T + a["t"] - a["dst"], axis=1)
    assert (res[a["inlier_mask"]] <= 6 * 0.005 + 1e-6).all()
