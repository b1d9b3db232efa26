"""Pins for oracle steps 1-3 (Eq. 1, Eq. 2, Def. 2) against things other than the oracle itself:
hand cases, closed forms, the App. E golden fixture, brute-force triangle counts (App. B), and an
independent numpy float64 evaluation of Eq. 1 that may differ only inside the near-threshold band."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import load_app_e, py_triangles, triangles_per_edge


# ------------------------------------------------------------------------------------------- Eq. 1
def test_compat_hand_cases():
    # both point pairs 1.0 m apart, τ = 0.01 → edge
    src = np.array([[0, 0, 0], [1, 0, 0]], np.float32)
    dst = np.array([[5, 5, 5], [5, 6, 5]], np.float32)
    C, e, _, _ = oracle.compat(src, dst, 0.01)
    assert e == 1 and C[0, 1] == 1 and C[1, 0] == 1 and C[0, 0] == 0
    # 1.0 m vs 1.5 m, τ = 0.1 → no edge
    dst2 = np.array([[0, 0, 0], [1.5, 0, 0]], np.float32)
    C, e, _, _ = oracle.compat(src, dst2, 0.1)
    assert e == 0 and C.sum() == 0


def test_compat_threshold_is_closed():
    # |1.0 - 1.5| = 0.5 exactly in float32: "≤ τ" is closed
    src = np.array([[0, 0, 0], [1, 0, 0]], np.float32)
    dst = np.array([[0, 0, 0], [1.5, 0, 0]], np.float32)
    assert oracle.compat(src, dst, 0.5)[1] == 1
    assert oracle.compat(src, dst, np.nextafter(np.float32(0.5), np.float32(0)))[1] == 0


def test_compat_exact_rigid_inliers_form_complete_graph():
    # distance preservation ⇒ complete subgraph over exact inliers
    inst = synth.generate(120, 1.0, (1, 1, 1), 0.0, seed=7)
    C, e, _, _ = oracle.compat(inst["src"], inst["dst"], 1e-4)
    assert e == 120 * 119 // 2
    assert (C + np.eye(120, dtype=np.uint8)).min() == 1


def test_compat_symmetry_monotonicity_equivariance():
    inst = synth.generate(150, 0.3, (1, 1, 1), 0.005, seed=11)
    C1, _, _, _ = oracle.compat(inst["src"], inst["dst"], 0.01)
    C2, _, _, _ = oracle.compat(inst["src"], inst["dst"], 0.02)
    assert (C1 == C1.T).all() and np.diag(C1).sum() == 0
    assert (C1 <= C2).all()  # S:175 τ-monotonicity
    perm = np.random.default_rng(0).permutation(150)
    Cp, _, _, _ = oracle.compat(inst["src"][perm], inst["dst"][perm], 0.01)
    assert (Cp == C1[np.ix_(perm, perm)]).all()  # S:176 permutation equivariance


def test_compat_matches_float64_definition_outside_band():
    # The real-number definition evaluated independently in float64 by numpy must agree with the
    # oracle's float32 decisions everywhere except inside the near-threshold band (reading r1).
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg)
    src64, dst64 = inst["src"].astype(np.float64), inst["dst"].astype(np.float64)
    a = np.linalg.norm(src64[:, None] - src64[None], axis=-1)
    b = np.linalg.norm(dst64[:, None] - dst64[None], axis=-1)
    d = np.abs(a - b)
    ref = (d <= np.float64(np.float32(cfg.tau))).astype(np.uint8)
    np.fill_diagonal(ref, 0)
    C, e, near, dis = oracle.compat(inst["src"], inst["dst"], cfg.tau)
    diff = np.argwhere(np.triu(C != ref, 1))
    assert len(diff) == dis
    for i, j in diff:
        band = 1e-6 + 4 * np.spacing(np.float32(max(a[i, j], b[i, j])))
        assert abs(d[i, j] - np.float32(cfg.tau)) <= band
    assert e == int(np.triu(C, 1).sum())


# ------------------------------------------------------------------------------------------- Eq. 2
def test_sc2_golden_fixture():
    g = load_app_e()
    G = oracle.sc2(g["C"])
    for (i, j), w in g["sc2"].items():
        assert G[i, j] == w and G[j, i] == w, (i, j)
    assert int((G > 0).sum()) == 2 * len(g["sc2"])  # no weight off the 15 edges
    for i, s in g["rowsum"].items():
        assert G[i].sum() == s
    assert len(oracle.brute_triangles(g["C"])) == g["triangles"] == len(py_triangles(g["C"]))


@pytest.mark.parametrize("density", [0.05, 0.2, 0.5])
@pytest.mark.parametrize("seed", range(4))
def test_sc2_equals_bruteforce_triangle_count(density, seed):
    # App. B / SPEC acceptance 1: Ĝ_ij = #3-cliques containing edge (i,j)
    n = 24 + 9 * seed
    C = synth.erdos_renyi(n, density, 100 * seed + int(density * 100))
    G = oracle.sc2(C)
    cnt = triangles_per_edge(C)
    for i, j in itertools.product(range(n), repeat=2):
        if i == j or not C[i, j]:
            assert G[i, j] == 0
        else:
            assert G[i, j] == cnt.get((min(i, j), max(i, j)), 0)
    tri = py_triangles(C)
    assert np.triu(G, 1).sum() == 3 * len(tri)  # Σ_{i<j} Ĝ_ij = 3T
    per_node = np.zeros(n, np.int64)
    for t in tri:
        per_node[list(t)] += 1
    assert (G.sum(1) == 2 * per_node).all()  # r_i = 2 t_i


def test_sc2_complete_graph_closed_form():
    n = 37
    C = (1 - np.eye(n)).astype(np.uint8)
    G = oracle.sc2(C)
    assert (G[~np.eye(n, dtype=bool)] == n - 2).all() and np.diag(G).sum() == 0


def test_sc2_edgeless_and_path():
    assert oracle.sc2(np.zeros((9, 9), np.uint8)).sum() == 0
    P = np.zeros((6, 6), np.uint8)
    for i in range(5):
        P[i, i + 1] = P[i + 1, i] = 1
    assert oracle.sc2(P).sum() == 0  # triangle-free


# ------------------------------------------------------------------------------------------- Def. 2
def test_o2_upper_triangle_and_half_sum():
    C = synth.erdos_renyi(40, 0.3, 5)
    G = oracle.sc2(C)
    O = oracle.o2(G)
    assert (np.tril(O) == 0).all()
    assert (np.triu(O, 1) == np.triu(G, 1)).all()
    assert 2 * O.sum() == G.sum()
    g = load_app_e()
    Of = oracle.o2(oracle.sc2(g["C"]))
    assert Of[6].sum() == 0  # highest index has no out-neighbours
