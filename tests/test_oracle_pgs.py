"""Pins for oracle steps 4-6 (Eq. 4 pivots, Alg. 1 PGS, canonical order): SPEC worked examples, the App. E
golden fixture, App. C unique assignment against brute-force triangles, closed forms on K_N, and the
linear-work counter of §3.4."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import load_app_e, py_triangles


def test_pivots_spec_example():
    # {(0,1):5, (0,2):3, (1,2):3}, K1 = 2 → (0,1) w5 then (0,2) w3
    G = np.zeros((3, 3), np.int32)
    for (i, j), w in {(0, 1): 5, (0, 2): 3, (1, 2): 3}.items():
        G[i, j] = G[j, i] = w
    assert oracle.select_pivots(G, 2).tolist() == [[0, 1, 5], [0, 2, 3]]
    assert len(oracle.select_pivots(G, 10)) == 3  # clamped to #positive edges


def test_pivots_complete_graph_all_ties():
    n = 12
    G = oracle.sc2((1 - np.eye(n)).astype(np.uint8))
    piv = oracle.select_pivots(G, 7)
    lex = [(i, j) for i in range(n) for j in range(i + 1, n)][:7]
    assert [tuple(p[:2]) for p in piv] == lex and (piv[:, 2] == n - 2).all()


def test_pivots_only_positive_weights():
    # a triangle-free path has edges but no positive SC² weight → no pivot (reading r5)
    C = np.zeros((5, 5), np.uint8)
    for i in range(4):
        C[i, i + 1] = C[i + 1, i] = 1
    assert len(oracle.select_pivots(oracle.sc2(C), 3)) == 0


def test_golden_fixture_pivots_and_cliques():
    g = load_app_e()
    G = oracle.sc2(g["C"])
    O = oracle.o2(G)
    piv = oracle.select_pivots(O, 2)
    assert [tuple(p) for p in piv] == g["pivot"]
    assert [tuple(p) for p in oracle.select_pivots(G, 2)] == g["pivot"]  # identical in both modes (r4)
    cl, _ = oracle.pgs(O, oracle.select_pivots(O, 1), 2)
    assert [tuple(c) for c in cl] == g["o2clique"]
    cl, _ = oracle.pgs(G, oracle.select_pivots(G, 1), 2)
    assert [tuple(c) for c in cl] == g["sc2clique"]


def _full_budget(C, mode):
    G = oracle.sc2(C)
    Gbar = oracle.o2(G) if mode == 0 else G
    n = C.shape[0]
    piv = oracle.select_pivots(Gbar, n * n)
    cl, chk = oracle.pgs(Gbar, piv, n)
    return piv, cl, chk


@pytest.mark.parametrize("density", [0.05, 0.2, 0.5])
@pytest.mark.parametrize("seed", range(3))
def test_unique_assignment_o2_equals_bruteforce(density, seed):
    # App. C, SPEC acceptance 2: O2, K1 = all edges, K2 = N → every triangle exactly once
    n = 20 + 11 * seed
    C = synth.erdos_renyi(n, density, 7 + seed * 13 + int(100 * density))
    piv, cl, chk = _full_budget(C, 0)
    got = sorted(tuple(c[:3]) for c in cl)
    assert got == sorted(py_triangles(C))
    assert chk == len(piv) * (n - 2)  # linear-work counter
    # Eq. 8 verification product on every emitted triple
    G = oracle.sc2(C)
    for i, j, z, s in cl:
        assert G[i, j] * G[i, z] * G[j, z] > 0 and s == G[i, j] + G[i, z] + G[j, z]


@pytest.mark.parametrize("seed", range(3))
def test_sc2_mode_finds_each_triangle_three_times(seed):
    # SPEC acceptance 3 (§3.3 "redundant TurboClique detection")
    C = synth.erdos_renyi(26, 0.3, 500 + seed)
    _, cl, _ = _full_budget(C, 1)
    tri = py_triangles(C)
    got = [tuple(c[:3]) for c in cl]
    assert len(got) == 3 * len(tri)
    assert all(got.count(t) == 3 for t in tri)
    assert sorted(set(tuple(c[:3]) for c in oracle.canonical(cl, dedup=True))) == sorted(tri)


def test_golden_full_budget():
    g = load_app_e()
    _, cl, _ = _full_budget(g["C"], 0)
    assert len(cl) == g["triangles"] and len(set(tuple(c[:3]) for c in cl)) == g["triangles"]
    _, cl, _ = _full_budget(g["C"], 1)
    assert len(cl) == 3 * g["triangles"]


def test_budget_bound_and_monotonicity():
    C = synth.erdos_renyi(30, 0.25, 99)
    O = oracle.o2(oracle.sc2(C))
    prev = -1
    for k1 in (1, 3, 10, 40):
        for k2 in (1, 2, 5):
            cl, _ = oracle.pgs(O, oracle.select_pivots(O, k1), k2)
            assert len(cl) <= k1 * k2
        cl2, _ = oracle.pgs(O, oracle.select_pivots(O, k1), 2)
        assert len(cl2) >= prev
        prev = len(cl2)


def test_k2_tie_keeps_lower_z():
    # K2 = 1 with two neighbours of equal S → lower z
    C = np.zeros((4, 4), np.uint8)
    for a, b in ((0, 1), (0, 2), (1, 2), (0, 3), (1, 3)):
        C[a, b] = C[b, a] = 1
    O = oracle.o2(oracle.sc2(C))
    cl, _ = oracle.pgs(O, np.array([[0, 1, O[0, 1]]], np.int32), 1)
    assert cl.tolist() == [[0, 1, 2, O[0, 1] + O[0, 2] + O[1, 2]]]


def test_canonical_order():
    cl = np.array([[0, 1, 2, 5], [0, 1, 3, 7], [0, 2, 3, 5], [0, 1, 4, 5]], np.int32)
    assert oracle.canonical(cl).tolist() == [[0, 1, 3, 7], [0, 1, 2, 5], [0, 1, 4, 5], [0, 2, 3, 5]]
