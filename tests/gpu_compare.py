"""Element-by-element comparison of one pair's CUDA intermediates with the oracle's trace.

Match criteria (BASELINE.json north_star):
  (i)   C bits, SC^2 weights, pivot set, clique set: bit-exact;
  (ii)  per clique, GPU (R, t) vs oracle (R, t): rotation within 1e-4 rad, translation within 1e-5 units;
  (iii) every GPU inlier count equals the oracle's recount on the GPU's float32 (R, t), bit-exact;
  (iv)  the final winner equals the oracle's.
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_2507_01439_b200._binding import I_CLIQUES, I_HYPS, I_PIVOTS, I_SC2, I_STATE

ROT_TOL_RAD = 1e-4
TRANS_TOL = 1e-5


def rot_angle_rad(Ra, Rb):
    d = np.linalg.norm(np.asarray(Ra, np.float64) - np.asarray(Rb, np.float64))
    return 2 * np.arcsin(min(1.0, d / (2 * np.sqrt(2))))


def gpu_trace(tr, pair=0):
    st = tr.intermediate(pair, I_STATE)
    cl = tr.intermediate(pair, I_CLIQUES)
    hy = tr.intermediate(pair, I_HYPS)
    valid = cl[:, 0] >= 0
    return {
        "state": st,
        "C": tr.bits(pair),
        "G": tr.intermediate(pair, I_SC2),
        "pivots": tr.intermediate(pair, I_PIVOTS),
        "cliques": cl[valid],
        "hyp_R": hy[valid, :9].reshape(-1, 3, 3),
        "hyp_t": hy[valid, 9:12],
        "hyp_count": hy[valid, 12].view(np.int32),
        "hyp_flag": hy[valid, 13].view(np.int32),
    }


def compare_pair(tr, pair, src, dst, tau, k1, k2, thr, result=None, check_graph=True, graph_mode=0):
    """Assert every match criterion for `pair` of the last call on context `tr`.  Returns stats."""
    ref = oracle.estimate(src, dst, tau, k1, k2, thr, graph_mode=graph_mode, trace=True)
    g = gpu_trace(tr, pair)
    n = src.shape[0]
    stats = {"n": n, "edges": ref["num_edges"], "near_edges": ref["near_edges"], "cliques": ref["num_cliques"]}
    # (i) graph
    assert g["state"]["edges"] == ref["num_edges"]
    if check_graph:
        diff = np.argwhere(g["C"] != ref["C"])
        assert len(diff) == 0, f"C differs at {len(diff)} entries, first {diff[:5].tolist()}"
        assert (g["G"] == ref["G"]).all(), f"SC2 differs at {int((g['G'] != ref['G']).sum())} entries"
    # (i) pivots: the same set; the GPU lists them in the oracle's (w desc, i, j) order unless > 8192 edges tie
    # at the cut (then lexicographically)
    rp = list(map(tuple, ref["pivots"].tolist()))
    gp = list(map(tuple, g["pivots"].tolist()))
    assert sorted(gp) == sorted(rp), f"pivots differ: {len(gp)} vs {len(rp)}"
    if rp:  # the order too, whenever the candidates at or above the cut weight fit the 8192-key sort
        alpha = min(w for _, _, w in rp)
        ncand = int((np.triu(ref["G"], 1) >= max(alpha, 1)).sum())
        if ncand <= 8192:
            assert gp == rp, "pivot order differs from (w desc, i asc, j asc)"
        stats["pivot_candidates"] = ncand
    # (i) cliques: the same set of (i, j, z, S)
    rc = sorted(map(tuple, ref["cliques"].tolist()))
    gc_order = np.lexsort(g["cliques"][:, ::-1].T)
    gcs = g["cliques"][gc_order]
    assert list(map(tuple, gcs.tolist())) == rc, "clique sets differ"
    # per-clique transforms and counts, aligned by (i, j, z)
    ro = np.lexsort(ref["cliques"][:, 2::-1].T)
    r_R, r_t = ref["hyp_R"][ro], ref["hyp_t"][ro]
    r_cnt, r_deg = ref["hyp_count"][ro], ref["hyp_degenerate"][ro]
    g_R, g_t = g["hyp_R"][gc_order], g["hyp_t"][gc_order]
    g_cnt, g_flag = g["hyp_count"][gc_order], g["hyp_flag"][gc_order]
    assert ((g_flag == 1) == (r_deg == 1)).all(), "degenerate flags differ"
    ok = g_flag == 0
    max_rot = max_tr = 0.0
    recount_mismatch = 0
    count_diff = 0
    for k in np.nonzero(ok)[0]:
        a = rot_angle_rad(g_R[k], r_R[k])
        b = float(np.abs(g_t[k].astype(np.float64) - r_t[k]).max())
        max_rot, max_tr = max(max_rot, a), max(max_tr, b)
        rc_ = oracle.count_inliers(src, dst, g_R[k], g_t[k], thr)
        recount_mismatch += int(rc_ != g_cnt[k])
        count_diff += int(g_cnt[k] != r_cnt[k])
    stats.update(max_rot_rad=max_rot, max_trans=max_tr, recount_mismatch=recount_mismatch, count_diff=count_diff,
                 hypotheses=int(ok.sum()))
    assert max_rot <= ROT_TOL_RAD and max_tr <= TRANS_TOL, stats
    assert recount_mismatch == 0, stats  # (iii)
    assert count_diff == 0, stats  # identical float32 (R, t) ⇒ identical counts
    # (iv) winner
    if result is not None:
        assert result["status"] == ref["status"], (result["status"], ref["status"])
        if ref["status"] == 0:
            assert tuple(result["clique"]) == tuple(ref["clique"]), (result["clique"], ref["clique"])
            assert result["inlier_count"] == ref["inlier_count"]
            assert result["clique_weight"] == ref["clique_weight"]
            assert rot_angle_rad(np.asarray(result["R"]).reshape(3, 3), ref["R"]) <= ROT_TOL_RAD
            assert np.abs(np.asarray(result["t"], np.float64) - ref["t"]).max() <= TRANS_TOL
        assert result["num_pivots"] == ref["num_pivots"]
        assert result["num_cliques"] == ref["num_cliques"]
        assert result["hypotheses_evaluated"] == ref["hypotheses_evaluated"]
        assert result["num_edges"] == ref["num_edges"]
    return stats
