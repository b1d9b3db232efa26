#!/usr/bin/env python3
"""Small workload for the checked build (TURBOREG_LIBRARY=lib/libturboreg_checked.so: device-side invariant
checks after every stage; compute-sanitizer is closed on the GPU pool) or compute-sanitizer: configs A and B
single pairs (the B pair runs the tcgen05 dense block with its mbarrier/TMEM pipeline and the bulk-copy
scoring ring), a 3-pair batch with host inputs (the pipelined sub-batch path), SC^2 mode with MAE ranking,
RANSAC, point resolution, the ranked list and a 2-rank split pair.  Exits non-zero on any result mismatch
against the plain call.  Not part of the product path.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2507_01439_b200 import TurboReg  # noqa: E402
from paper_2507_01439_b200.split import emulate_split  # noqa: E402


def main():
    ok = True
    for key, n in (("A", None), ("B", 2000)):
        cfg = synth.CONFIGS[key]
        inst = synth.workload_instance(cfg, pair=1, n=n)
        nn = inst["src"].shape[0]
        tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn, max_batch=3)
        tr.set_option("heavy_min_rows", 1)
        r = tr.register(inst["src"], inst["dst"])
        ok &= r["status"] == 0
        off = np.array([0, nn, 2 * nn], np.int64)
        res = tr.register_batch(np.concatenate([inst["src"]] * 3), np.concatenate([inst["dst"]] * 3), off,
                                np.full(3, nn, np.int32))
        ok &= all(tuple(x["clique"]) == tuple(r["clique"]) for x in res)
        ok &= len(tr.ranked_hypotheses(0, "in", top_k=4)) == 4
        tr.ransac(inst["src"], inst["dst"], 64, seed=3)
        tr.point_resolution(inst["src"])
        tr.close()
        t2 = TurboReg(cfg.tau, min(cfg.k1, 500), cfg.k2, cfg.inlier_threshold, max_n=nn, graph_mode=1, rank_metric="mae")
        ok &= t2.register(inst["src"], inst["dst"])["status"] == 0
        t2.close()
        engines = [TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=nn) for _ in range(2)]
        s = emulate_split(engines, inst["src"], inst["dst"])
        ok &= tuple(s["clique"]) == tuple(r["clique"]) and s["inlier_count"] == r["inlier_count"]
        for e in engines:
            e.close()
        print(key, "ok" if ok else "MISMATCH", flush=True)
    if "--full" in sys.argv:  # BASELINE-size pairs of configs C and D, a 4-pair batch, 1100 pairs, ER graphs
        for key in ("C", "D"):
            cfg = synth.CONFIGS[key]
            inst = synth.workload_instance(cfg, pair=2)
            tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=cfg.n, max_batch=4)
            r = tr.register(inst["src"], inst["dst"])
            off = np.arange(4, dtype=np.int64) * cfg.n
            res = tr.register_batch(np.concatenate([inst["src"]] * 4), np.concatenate([inst["dst"]] * 4), off,
                                    np.full(4, cfg.n, np.int32))
            ok &= r["status"] == 0 and all(tuple(x["clique"]) == tuple(r["clique"]) for x in res)
            print(key, "ok" if ok else "MISMATCH", flush=True)
            tr.close()
        # 1100 pairs: beyond the shared-memory tile table (1024 pairs), the dynamically scheduled tensor-core
        # block walks the global table across all of them
        cfg = synth.CONFIGS["E"]
        nb, n = 1100, 2000
        insts = [synth.workload_instance(cfg, pair=p, n=n) for p in range(nb)]
        tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n, max_batch=nb)
        res = tr.register_batch(np.concatenate([x["src"] for x in insts]), np.concatenate([x["dst"] for x in insts]),
                                np.arange(nb, dtype=np.int64) * n, np.full(nb, n, np.int32))
        ok &= bool((res["status"] == 0).all())
        for p in (0, 517, 1099):
            r = tr.register(insts[p]["src"], insts[p]["dst"])
            ok &= tuple(r["clique"]) == tuple(res[p]["clique"]) and r["inlier_count"] == res[p]["inlier_count"]
        tr.close()
        print("E x1100 ok" if ok else "E x1100 MISMATCH", flush=True)
        tr = TurboReg(0.01, 200, 4, 0.1, max_n=300)
        for dens in (0.05, 0.2, 0.5):
            tr.pgs_from_adjacency(synth.erdos_renyi(300, dens, seed=int(dens * 100)))
        print("ER ok", flush=True)
    from paper_2507_01439_b200._binding import library_path

    print("library", library_path(), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
