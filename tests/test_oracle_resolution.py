"""Oracle pins for the point-cloud resolution of the τ initialisation (τ = 0.25·pr, P:322, P:623-624;
SURVEY.md §8(f) row 3): SPEC's worked examples and a library nearest-neighbour routine
(scipy cKDTree, float64) on random clouds, within float32 rounding."""
import numpy as np
import pytest

import oracle


def test_spec_examples():
    lattice = np.stack([np.arange(10.0), np.zeros(10), np.zeros(10)], 1)  # unit-spaced 1-D lattice → 1.0
    assert oracle.point_resolution(lattice) == 1.0
    assert oracle.point_resolution(np.array([[0.0, 0, 0], [0.5, 0, 0]])) == 0.5  # two points 0.5 apart
    assert oracle.point_resolution(np.zeros((1, 3))) == -1.0  # fewer than 2 points


@pytest.mark.parametrize("n,seed", [(2, 0), (7, 1), (500, 2), (3001, 3)])
def test_matches_kdtree_median(n, seed):
    spatial = pytest.importorskip("scipy.spatial")
    rng = np.random.default_rng(seed)
    xyz = rng.uniform(-1.5, 1.5, size=(n, 3)).astype(np.float32)
    d, _ = spatial.cKDTree(xyz.astype(np.float64)).query(xyz.astype(np.float64), k=2)
    ref = np.sort(d[:, 1])[(n - 1) // 2]  # lower median (reading r22)
    got = oracle.point_resolution(xyz)
    assert abs(got - ref) <= 4e-7 * max(ref, 1e-30) + 1e-12


def test_duplicates_and_order():
    xyz = np.array([[0, 0, 0], [0, 0, 0], [1, 0, 0], [3, 0, 0]], np.float32)  # nn: 0, 0, 1, 2 → lower median 0
    assert oracle.point_resolution(xyz) == 0.0
    perm = np.random.default_rng(0).permutation(4)
    assert oracle.point_resolution(xyz[perm]) == 0.0
