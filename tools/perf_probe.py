#!/usr/bin/env python3
"""Per-kernel timing probe (CUDA events inside libturboreg) for tuning: runs the bench workload shape under a
few option settings and prints ms per kernel per pair.  Not part of the product path.

    python tools/perf_probe.py [--pairs 64] [--cfg E] [--opt sc2_path=1 --opt heavy_min_rows=100000]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_01439_b200 import RESULT_DTYPE, TurboReg  # noqa: E402


def run(cfg, pairs, opts, reps=3, n=None, graph_mode=0, rank_metric="in", hyp_errors=False):
    n = n or cfg.n
    src = np.concatenate([synth.workload_instance(cfg, pair=p, n=n)["src"] for p in range(pairs)])
    dst = np.concatenate([synth.workload_instance(cfg, pair=p, n=n)["dst"] for p in range(pairs)])
    off = (np.arange(pairs) * n).astype(np.int64)
    nn = np.full(pairs, n, np.int32)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    sd, dd = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    out = torch.zeros(pairs * RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n, max_batch=pairs, kernel_timing=True,
                  graph_mode=graph_mode, rank_metric=rank_metric, hyp_errors=hyp_errors)
    for k, v in opts.items():
        tr.set_option(k, v)
    for _ in range(2):
        tr.register_batch(sd, dd, off, nn, out=out, stream=s.cuda_stream)
    torch.cuda.synchronize()
    tr.profile_begin()
    for _ in range(reps):
        tr.register_batch(sd, dd, off, nn, out=out, stream=s.cuda_stream)
    torch.cuda.synchronize()
    prof = tr.profile_end()
    res = out.cpu().numpy().view(RESULT_DTYPE)
    per = {k: round(v[0] / reps / pairs * 1000, 3) for k, v in prof.items() if v[1]}
    per["TOTAL_us_per_pair"] = round(sum(per.values()), 2)
    per["status_ok"] = int((res["status"] == 0).sum())
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=64)
    ap.add_argument("--cfg", default="E")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--variants", default="")
    ap.add_argument("--graph-mode", type=int, default=0)
    ap.add_argument("--rank-metric", default="in", choices=["in", "mae", "mse"])
    ap.add_argument("--hyp-errors", action="store_true")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.cfg]
    variants = [dict(kv.split("=") for kv in args.opt)]
    if args.variants:
        variants = [dict(kv.split("=") for kv in v.split(",") if kv) for v in args.variants.split(";")]
    for v in variants:
        opts = {k: int(x) for k, x in v.items()}
        print(json.dumps({"cfg": args.cfg, "opts": opts, "graph_mode": args.graph_mode,
                          "rank_metric": args.rank_metric, "hyp_errors": args.hyp_errors,
                          "us_per_pair": run(cfg, args.pairs, opts, n=args.n, graph_mode=args.graph_mode,
                                             rank_metric=args.rank_metric, hyp_errors=args.hyp_errors)}))


if __name__ == "__main__":
    main()
