"""The largest supported pair (n = max_n = 32768: 1024 words per bit row, the 32-word-per-lane kernels)
checked on sampled outputs the oracle computes one by one, and by properties that hold at any size
(Ĝ = popcount of row AND, top-K1 / top-K2 orders, triangle and weight identities).  Needs a B200."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_compare import rot_angle_rad

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def run():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import TurboReg

    cfg = synth.CONFIGS["C"]
    n = 32768
    inst = synth.workload_instance(cfg, pair=3, n=n)
    tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n)
    res = tr.register(inst["src"], inst["dst"])
    return cfg, n, inst, tr, res


def _rows(tr, n):
    from paper_2507_01439_b200._binding import I_BITS, I_STATE

    W = tr.intermediate(0, I_STATE)["W"]
    return tr.intermediate(0, I_BITS).reshape(n, W)


def _bit(rows, i, j):
    return (rows[i, j >> 5] >> np.uint32(j & 31)) & 1


def test_compat_sampled(run):
    cfg, n, inst, tr, res = run
    rows = _rows(tr, n)
    rng = np.random.default_rng(11)
    pairs = rng.integers(0, n, (4000, 2))
    # plus pairs near the threshold (chosen in float64, decided by the oracle's float32 tree)
    s, d = inst["src"].astype(np.float64), inst["dst"].astype(np.float64)
    a = rng.integers(0, n, 200000)
    b = rng.integers(0, n, 200000)
    dlt = np.abs(np.linalg.norm(s[a] - s[b], axis=1) - np.linalg.norm(d[a] - d[b], axis=1))
    near = np.argsort(np.abs(dlt - cfg.tau))[:2000]
    pairs = np.concatenate([pairs, np.stack([a[near], b[near]], 1)])
    for i, j in pairs:
        if i == j:
            continue
        C, _, _, _ = oracle.compat(inst["src"][[i, j]], inst["dst"][[i, j]], cfg.tau)
        assert _bit(rows, i, j) == C[0, 1] and _bit(rows, j, i) == C[1, 0], (i, j)


def test_sc2_edges_and_pivots(run):
    from paper_2507_01439_b200._binding import I_EDGES, I_PIVOTS

    cfg, n, inst, tr, res = run
    rows = _rows(tr, n)
    rp, E = tr.intermediate(0, I_EDGES)
    assert rp[0] == 0 and rp[-1] == len(E) == int(res["num_edges"])
    jj = (E >> 16).astype(np.int64)
    ww = (E & 0xFFFF).astype(np.int64)
    rng = np.random.default_rng(12)
    for i in rng.integers(0, n, 300):  # row i's list = the set bits of U_i, in increasing j
        bits = np.unpackbits(rows[i].view(np.uint8), bitorder="little")[:n]
        up = np.nonzero(bits)[0]
        up = up[up > i]
        assert (jj[rp[i]:rp[i + 1]] == up).all()
    pop = np.vectorize(lambda x: bin(int(x)).count("1"))
    for e in rng.integers(0, len(E), 3000):  # Ĝ_ij = |N(i) ∩ N(j)|
        i = int(np.searchsorted(rp, e, side="right") - 1)
        j = int(jj[e])
        assert ww[e] == int(pop(rows[i] & rows[j]).sum())
    # pivots: the first K1 positive edges by (w desc, i asc, j asc)
    ii = np.repeat(np.arange(n), np.diff(rp))
    pos = ww > 0
    order = np.lexsort((jj[pos], ii[pos], -ww[pos]))[: cfg.k1]
    want = np.stack([ii[pos][order], jj[pos][order], ww[pos][order]], 1)
    got = tr.intermediate(0, I_PIVOTS)
    assert sorted(map(tuple, got.tolist())) == sorted(map(tuple, want.tolist()))


def test_cliques_hypotheses_winner(run):
    from paper_2507_01439_b200._binding import I_CLIQUES, I_EDGES, I_HYPS, I_PIVOTS

    cfg, n, inst, tr, res = run
    rows = _rows(tr, n)
    rp, E = tr.intermediate(0, I_EDGES)
    jj = (E >> 16).astype(np.int64)
    ww = (E & 0xFFFF).astype(np.int64)

    def w(i, j):
        i, j = min(i, j), max(i, j)
        k = rp[i] + np.searchsorted(jj[rp[i]:rp[i + 1]], j)
        assert jj[k] == j
        return int(ww[k])

    piv = tr.intermediate(0, I_PIVOTS)
    cl = tr.intermediate(0, I_CLIQUES).reshape(-1, cfg.k2, 4)
    rng = np.random.default_rng(13)
    for p in rng.choice(len(piv), 60, replace=False):  # top-K2 of each sampled pivot, recomputed
        i, j, wij = map(int, piv[p])
        ri = np.unpackbits(rows[i].view(np.uint8), bitorder="little")[:n].astype(bool)
        rj = np.unpackbits(rows[j].view(np.uint8), bitorder="little")[:n].astype(bool)
        z = np.nonzero(ri & rj)[0]
        z = z[z > j]
        S = np.array([wij + w(i, k) + w(j, k) for k in z], np.int64)
        o = np.lexsort((z, -S))[: cfg.k2]
        want = [(i, j, int(z[k]), int(S[k])) for k in o]
        got = [tuple(c) for c in cl[p].tolist() if c[0] >= 0]
        assert got == want
    hy = tr.intermediate(0, I_HYPS)
    flat = tr.intermediate(0, I_CLIQUES)
    valid = np.nonzero((flat[:, 0] >= 0) & (hy[:, 13].view(np.int32) == 0))[0]
    for s in rng.choice(valid, 80, replace=False):  # Kabsch and the inlier count against the oracle
        i, j, z, _ = flat[s]
        fit = oracle.kabsch(inst["src"][[i, j, z]], inst["dst"][[i, j, z]])
        R, t = hy[s, :9].reshape(3, 3), hy[s, 9:12]
        assert rot_angle_rad(R, fit[0]) <= 1e-4 and np.abs(t - fit[1]).max() <= 1e-5
        assert oracle.count_inliers(inst["src"], inst["dst"], R, t, cfg.inlier_threshold) == hy[s, 12].view(np.int32)
    # the winner is the (count desc, S desc, ijz asc) maximum over the GPU's own hypotheses
    cnt = hy[valid, 12].view(np.int32).astype(np.int64)
    S = hy[valid, 14].view(np.int32).astype(np.int64)
    best = valid[np.lexsort((flat[valid, 2], flat[valid, 1], flat[valid, 0], -S, -cnt))[0]]
    assert tuple(flat[best, :3]) == tuple(res["clique"]) and res["status"] == 0
    assert synth.rotation_error_deg(res["R"].reshape(3, 3), inst["R"]) <= 5
