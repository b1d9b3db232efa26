"""NEXT(1) exchange choreography on CPU (gloo, world sizes 2 and 3): paper_2507_01439_b200.split.register_split
drives a stand-in engine that follows the library's split contract (include/turboreg.h "NEXT(1)") with the
oracle's trace: each rank contributes only its share of C's words (the compat block-row-pair partition of
turboreg_compat.cuh), of the O2 edge words and of the pivots; the collectives must rebuild the full arrays
and the merged record must equal the single-rank oracle result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_2507_01439_b200._binding import RESULT_DTYPE, SPLIT_BITS, SPLIT_EDGES, SPLIT_RESULT
from paper_2507_01439_b200.sharding import shard_range

CFG = synth.CONFIGS["A"]


def _words(C):
    n = C.shape[0]
    T = (n + 31) // 32
    pad = np.zeros((n, T * 32), np.uint8)
    pad[:, :n] = C
    return np.packbits(pad, axis=1, bitorder="little").view(np.uint32).astype(np.int64), T


class MockEngine:
    """The split contract, computed from the oracle: phase outputs restricted to this rank's share."""

    def __init__(self, inst):
        self.ref = oracle.estimate(inst["src"], inst["dst"], CFG.tau, CFG.k1, CFG.k2, CFG.inlier_threshold,
                                   trace=True)
        self.words, self.T = _words(self.ref["C"])
        G = self.ref["G"]
        up = np.argwhere(np.triu(self.ref["C"], 1) > 0)  # row-major (i, j), i < j: the compact O2 rows
        self.edge_words = ((up[:, 1].astype(np.int64) << 16) | G[up[:, 0], up[:, 1]]).astype(np.int64)

    def split_begin(self, src, dst, rank, world, stream=None):
        n = src.shape[0]
        if n < 3:
            return 2
        self.rank, self.world = rank, world
        T = self.T
        bpp = (T + 1) // 2
        b0, b1 = shard_range(bpp, world, rank)
        I = np.arange(n)[:, None] // 32
        J = np.arange(T)[None, :]
        imin = np.minimum(I, J)
        b = np.minimum(imin, T - 1 - imin)  # tile (min(I,J), max(I,J)) belongs to block-row pair b
        own = (b >= b0) & (b < b1)
        self.bits = torch.from_numpy(np.where(own, self.words, 0).astype(np.int32).reshape(-1).copy())
        return 0

    def split_tensor(self, which, count=None):
        if which == SPLIT_BITS:
            return self.bits
        if which == SPLIT_EDGES:
            return self.edges[:count]
        return self.rec

    def split_sc2(self, stream=None):
        assert (self.bits.numpy().astype(np.int64) & 0xffffffff == self.words.reshape(-1)).all(), "bits not rebuilt"
        E = len(self.edge_words)
        own = (np.arange(E) % self.world) == self.rank  # any disjoint cover: each word written by one rank
        self.edges = torch.from_numpy(np.where(own, self.edge_words, 0).astype(np.int32).copy())
        return E

    def split_search(self, stream=None):
        assert (self.edges.numpy().astype(np.int64) == self.edge_words).all(), "edges not rebuilt"
        ref = self.ref
        piv = [tuple(p[:2]) for p in ref["pivots"].tolist()]
        P = len(piv)
        p0, p1 = shard_range(P, self.world, self.rank)
        mine = set(piv[p0:p1])
        rec = np.zeros(1, RESULT_DTYPE)[0]
        best = None
        ncl = nev = 0
        for k, c in enumerate(ref["cliques"].tolist()):
            if (c[0], c[1]) not in mine:
                continue
            ncl += 1
            if ref["hyp_degenerate"][k]:
                continue
            nev += 1
            key = (-int(ref["hyp_count"][k]), -c[3], tuple(c[:3]))
            if best is None or key < best[0]:
                best = (key, k)
        rec["num_pivots"], rec["num_cliques"], rec["hypotheses_evaluated"] = P, ncl, nev
        rec["num_edges"] = len(self.edge_words)
        rec["clique"] = (-1, -1, -1)
        rec["status"] = 5
        if best is not None:
            k = best[1]
            c = ref["cliques"][k]
            rec["status"], rec["inlier_count"], rec["clique"], rec["clique_weight"] = 0, ref["hyp_count"][k], c[:3], c[3]
            rec["R"], rec["t"] = ref["hyp_R"][k].reshape(9), ref["hyp_t"][k]
        self.rec = torch.from_numpy(np.frombuffer(rec.tobytes(), np.uint8).copy())

    def split_merge(self, parts, world, stream=None):
        recs = parts.numpy().view(RESULT_DTYPE)
        ok = [r for r in recs if r["status"] == 0]
        best = min(ok, key=lambda r: (-int(r["inlier_count"]), -int(r["clique_weight"]),
                                      tuple(int(x) for x in r["clique"]))) if ok else recs[0]
        out = {k: (best[k].copy() if np.ndim(best[k]) else best[k].item()) for k in RESULT_DTYPE.names}
        out["num_cliques"] = int(recs["num_cliques"].sum())
        out["hypotheses_evaluated"] = int(recs["hypotheses_evaluated"].sum())
        if not ok:
            out["status"] = 5
        return out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2507_01439_b200.split import register_split

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = synth.workload_instance(CFG, pair=7)
    res = register_split(MockEngine(inst), inst["src"], inst["dst"])
    q.put((rank, {k: (np.asarray(v).tolist()) for k, v in res.items()}))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_split_choreography_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inst = synth.workload_instance(CFG, pair=7)
    ref = oracle.estimate(inst["src"], inst["dst"], CFG.tau, CFG.k1, CFG.k2, CFG.inlier_threshold)
    for rank, res in got:
        assert res["status"] == ref["status"] == 0
        assert tuple(res["clique"]) == tuple(ref["clique"])
        for k in ("inlier_count", "clique_weight", "num_pivots", "num_cliques", "hypotheses_evaluated", "num_edges"):
            assert res[k] == ref[k], (rank, k, res[k], ref[k])
        assert np.abs(np.asarray(res["R"], np.float32).reshape(3, 3) - ref["R"]).max() == 0


def test_split_too_few_points_gloo_free():
    """A pair with n < 3 returns its status from phase 1 without any exchange."""
    inst = synth.workload_instance(CFG, pair=7)
    eng = MockEngine(inst)
    assert eng.split_begin(inst["src"][:2], inst["dst"][:2], 0, 2) == 2
