#!/usr/bin/env python3
"""End-to-end (pinned host inputs -> host results) time per batch through turboreg_register_batch, for a
set of library options.  usage: python tools/e2e_probe.py [--pairs 203] [--variants "pipeline_host_inputs=0;..."]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def main():
    import torch

    from paper_2507_01439_b200 import TurboReg

    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=203)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--variants", default="pipeline_host_inputs=1;pipeline_host_inputs=0")
    args = ap.parse_args()
    cfg = synth.CONFIGS["E"]
    n = cfg.n
    src = np.concatenate([synth.workload_instance(cfg, pair=p)["src"] for p in range(args.pairs)])
    dst = np.concatenate([synth.workload_instance(cfg, pair=p)["dst"] for p in range(args.pairs)])
    src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
    off = (np.arange(args.pairs) * n).astype(np.int64)
    nn = np.full(args.pairs, n, np.int32)
    for v in args.variants.split(";"):
        opts = {k: int(x) for k, x in (kv.split("=") for kv in v.split(",") if kv)}
        tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n, max_batch=args.pairs)
        for k, x in opts.items():
            tr.set_option(k, x)
        for _ in range(3):
            tr.register_batch(src_p, dst_p, off, nn)
        ts = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tr.register_batch(src_p, dst_p, off, nn)
            ts.append(time.perf_counter() - t0)
        tr.close()
        print(json.dumps({"opts": opts, "ms_median": 1000 * float(np.median(ts)), "ms_min": 1000 * min(ts),
                          "reg_per_s": args.pairs / float(np.median(ts))}))


if __name__ == "__main__":
    main()
