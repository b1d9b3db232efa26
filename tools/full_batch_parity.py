#!/usr/bin/env python3
"""Every pair of the bench's 1623-pair batch (or --cfg A-D: --pairs pairs of that config) against the oracle on its result record (status, T*'s clique,
inlier count, S, pivots, cliques, hypotheses, edges, R and t within the parity tolerances): the batch runs once
on the GPU exactly as bench.py launches it, the oracle runs in a pool of host processes (≈ 4 min on 16
cores).  Evidence, not part of the test suite.  usage: python tools/full_batch_parity.py > out.txt"""
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from tests.test_gpu_bench_batch import _oracle_record  # noqa: E402
from tests.gpu_compare import ROT_TOL_RAD, TRANS_TOL, rot_angle_rad  # noqa: E402

KEYS = ("status", "inlier_count", "clique_weight", "num_pivots", "num_cliques", "hypotheses_evaluated", "num_edges")


def _oracle_record_cfg(args):
    """The oracle's result record for pair `pair` of config `key` (spawn-pool worker)."""
    key, pair = args
    import oracle
    import synth

    cfg = synth.CONFIGS[key]
    inst = synth.workload_instance(cfg, pair=pair)
    r = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)
    return {**{k: int(r[k]) for k in KEYS}, "clique": tuple(int(x) for x in r["clique"]),
            "R": np.asarray(r["R"], np.float64).reshape(3, 3), "t": np.asarray(r["t"], np.float64)}


def main():
    import argparse

    import torch

    import synth
    from paper_2507_01439_b200 import RESULT_DTYPE, TurboReg

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="E", help="E = the bench batch (1623 pairs); A-D: --pairs pairs of that config")
    ap.add_argument("--pairs", type=int, default=64)
    args = ap.parse_args()
    if args.cfg == "E":
        cfg, pairs, n = bench.CFG, bench.SWEEP, bench.CFG.n
        src, dst, _ = bench.make_inputs(0, pairs)
        density = bench.MAX_DENSITY
    else:
        cfg, pairs = synth.CONFIGS[args.cfg], args.pairs
        insts = [synth.workload_instance(cfg, pair=p) for p in range(pairs)]
        n = insts[0]["src"].shape[0]
        src = np.concatenate([x["src"] for x in insts])
        dst = np.concatenate([x["dst"] for x in insts])
        density = 1.0
    tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n, max_batch=pairs, max_density=density)
    out = torch.zeros(pairs * RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    sd, dd = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    tr.register_batch(sd, dd, (np.arange(pairs) * n).astype(np.int64), np.full(pairs, n, np.int32), out=out)
    torch.cuda.synchronize()
    res = out.cpu().numpy().view(RESULT_DTYPE).copy()
    t0 = time.time()
    workers = len(os.sched_getaffinity(0))
    with mp.get_context("spawn").Pool(workers) as pool:
        if args.cfg == "E":
            refs = pool.map(_oracle_record, range(pairs), chunksize=4)
        else:
            refs = pool.map(_oracle_record_cfg, [(args.cfg, p) for p in range(pairs)])
    bad = []
    max_rot = max_tr = 0.0
    for p, ref in enumerate(refs):
        got = res[p]
        diff = [k for k in KEYS if int(got[k]) != ref[k]]
        if tuple(int(x) for x in got["clique"]) != ref["clique"]:
            diff.append("clique")
        a = rot_angle_rad(np.asarray(got["R"]).reshape(3, 3), ref["R"])
        b = float(np.abs(np.asarray(got["t"], np.float64) - ref["t"]).max())
        max_rot, max_tr = max(max_rot, a), max(max_tr, b)
        if a > ROT_TOL_RAD or b > TRANS_TOL:
            diff.append("transform")
        if diff:
            bad.append((p, diff))
    what = "bench batch" if args.cfg == "E" else f"config {args.cfg} ({cfg.name})"
    print(f"{what}: {pairs} pairs (N = {n}, K1 = {cfg.k1}, K2 = {cfg.k2}), one register_batch call")
    print(f"oracle: {workers} host processes, {time.time() - t0:.0f} s")
    print(f"fields compared per pair: {', '.join(KEYS)}, clique; R within {ROT_TOL_RAD} rad, t within {TRANS_TOL}")
    print(f"pairs identical to the oracle: {pairs - len(bad)} / {pairs}")
    print(f"max rotation difference {max_rot:.3g} rad, max translation difference {max_tr:.3g}")
    print(f"status 0 (GPU): {int((res['status'] == 0).sum())} / {pairs}")
    for p, d in bad[:20]:
        print("  mismatch", p, d)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
