"""Oracle pins for the equal-budget 3-point RANSAC baseline.

The sampler is the counter-based SplitMix64 generator (Steele, Lea & Flood, "Fast splittable pseudorandom
number generators", OOPSLA 2014; reference implementation splitmix64.c by S. Vigna), pinned to its
published output stream; the triple construction is pinned by its distribution (distinct, sorted,
uniform over indices, every triple reachable); the fit/score plumbing by planted data."""
import itertools

import numpy as np

import oracle
import synth


def test_splitmix64_matches_the_published_stream():
    # splitmix64.c seeded with state 0: the first three outputs
    assert [oracle.splitmix64(0, k) for k in range(3)] == [
        0xE220A8397B1DCDAF,
        0x6E789E6AA1B965F4,
        0x06C45D188009454F,
    ]


def test_triples_are_sorted_distinct_and_in_range():
    for n in (3, 4, 7, 500):
        for k in range(300):
            t = oracle.ransac_triple(123, k, n)
            assert 0 <= t[0] < t[1] < t[2] < n
    assert {oracle.ransac_triple(9, k, 3) for k in range(20)} == {(0, 1, 2)}


def test_triples_cover_all_subsets_uniformly():
    n, m = 10, 24000
    seen = {}
    freq = np.zeros(n)
    for k in range(m):
        t = oracle.ransac_triple(2024, k, n)
        seen[t] = seen.get(t, 0) + 1
        freq[list(t)] += 1
    assert set(seen) == set(itertools.combinations(range(n), 3))  # every 3-subset reachable
    expect = 3 * m / n  # each index in 3/n of the triples
    assert np.all(np.abs(freq - expect) < 5 * np.sqrt(expect))
    cnt = np.array(list(seen.values()), float)  # 120 subsets, m/120 = 200 each
    assert abs(cnt.mean() - m / 120) < 1e-9 and cnt.min() > 140 and cnt.max() < 260


def test_seed_changes_the_stream_and_is_reproducible():
    a = [oracle.ransac_triple(1, k, 1000) for k in range(50)]
    b = [oracle.ransac_triple(2, k, 1000) for k in range(50)]
    assert a != b and a == [oracle.ransac_triple(1, k, 1000) for k in range(50)]


def test_exact_correspondences_are_all_inliers():
    # noise-free, outlier-free correspondences: any non-degenerate triple recovers T, so the count is N
    g = synth.generate(300, 1.0, (2.0, 2.0, 2.0), 0.0, seed=77)
    r = oracle.ransac(g["src"], g["dst"], 20, seed=5, inlier_threshold=1e-3)
    assert r["status"] == 0 and r["inlier_count"] == 300
    assert synth.rotation_error_deg(r["R"].astype(np.float64), g["R"]) < 0.05  # float32-rounded points


def test_each_slot_is_its_triple_fitted_and_scored():
    cfg = synth.CONFIGS["A"]
    inst = synth.workload_instance(cfg, pair=3)
    r = oracle.ransac(inst["src"], inst["dst"], 60, seed=11, inlier_threshold=cfg.inlier_threshold, trace=True)
    best = None
    for k in range(60):
        tri = tuple(int(x) for x in r["cliques"][k, :3])
        assert tri == oracle.ransac_triple(11, k, inst["src"].shape[0])
        if r["hyp_degenerate"][k]:
            continue
        P = inst["src"][list(tri)].astype(np.float64)
        Q = inst["dst"][list(tri)].astype(np.float64)
        R, t = oracle.kabsch(P, Q)
        c = oracle.count_inliers(inst["src"], inst["dst"], R.astype(np.float32), t.astype(np.float32),
                                 cfg.inlier_threshold)
        assert c == r["hyp_count"][k]
        key = (-c, tri)
        best = key if best is None or key < best else best
    assert r["inlier_count"] == -best[0] and r["clique"] == best[1]  # (count desc, ijz asc)
