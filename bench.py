#!/usr/bin/env python3
"""Benchmark: registrations/sec at N=5000 with 1K TurboCliques (K1=1000, K2=2) on 1/2/4/8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sweep 1623 | --pairs P] [--impl reference]

Workload (BASELINE.json configs[4]): the 1623-pair 3DMatch-shaped sweep (configs[1] parameters,
N=5000, K1=1000, K2=2), sharded over the N ranks (rank r registers pairs shard_range(1623, N, r)): strong
scaling, the same total work at every N.  `--pairs P` instead gives every rank its own P pairs (weak
scaling).  One step = one pass of the whole hot path (compat → SC^2 → pivots → PGS → Kabsch → scoring →
argmax) over the rank's pairs in one batched call, on the library's default path (CUDA-graph replay, the
sparse-row SC^2 kernel on a side stream).  Inputs are resident in HBM when the timed region starts; L2 is
flushed (256 MiB write) before every timed step.  Timing is CUDA events on the launching stream with a
barrier + synchronize on both sides, max over ranks; rank 0 prints one JSON line.  Per-kernel times come
from a separate pass over the same batch with per-kernel CUDA events (direct launches, one stream).

`--gpus N` with no torchrun environment re-launches itself under `torch.distributed.run` with N ranks (one
per GPU, NCCL).  `--impl reference` times the CPU oracle (oracle/, the only other place this script
executes it) on the host cores, a bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "registrations/s"
CFG = synth.CONFIGS["E"]
SWEEP = synth.BATCH_PAIRS  # 1623: the 3DMatch pair count, configs[4]
MAX_DENSITY = 0.125  # per-pair edge capacity: 1/8 of all N(N-1)/2 pairs (config E measures 4.35 %)
L2_FLUSH_BYTES = 256 << 20
SMS = 148
MMA_FP4 = 1  # dense SC^2 block as tcgen05.mma kind::mxf4 (the library default); 0 = kind::i8


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "_fallback": True}


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for k, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class NvmlClockSampler:
    """The same record from NVML, polled every 5 ms by a thread (nvidia-smi's start-up can miss a short
    timed region).  Reasons: NVML clock-event bits hw_slowdown 0x8, sw_thermal 0x20, hw_thermal 0x40,
    sw_power_cap 0x4."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        self.sm, self.reasons = [], set()
        self.run = False

    def _poll(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while self.run:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = int(get_reasons(self.h))
                for k, b in self.BITS.items():
                    if r & b:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        self.run = True
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()

    def stop(self):
        self.run = False
        self.t.join(timeout=2)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


def clock_sampler(index):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


# ------------------------------------------------------------------------------------------ workload
def make_inputs(first, pairs, n=None):
    """Global pairs [first, first + pairs) of the configs[4] sweep (pair p: seed CFG.seed + p)."""
    n = n or CFG.n
    src = np.empty((pairs * n, 3), np.float32)
    dst = np.empty((pairs * n, 3), np.float32)
    gts = []
    for k in range(pairs):
        inst = synth.workload_instance(CFG, pair=first + k, n=n)
        src[k * n:(k + 1) * n] = inst["src"]
        dst[k * n:(k + 1) * n] = inst["dst"]
        gts.append((inst["R"], inst["t"]))
    return src, dst, gts


def algorithmic_work(tr, res, pairs):
    """Algorithmic work of the last call, summed over its pairs: compat pair tests, the
    dense tensor-core block's operations, scoring residual tests, O2 edges, bytes of the memory passes."""
    from paper_2507_01439_b200._binding import I_STATE

    tests = mma_ops = mma_useful = edges = deg_bytes = expand_bytes = 0
    for p in range(pairs):
        st = tr.intermediate(p, I_STATE)
        n, W, h = st["n"], st["W"], st["heavy_h"]
        tests += n * (n - 1) // 2
        edges += st["edges"]
        deg_bytes += 4 * n * W + 8 * n  # every bit row read, degree + upper degree written
        if h:  # upper 128 x TN tiles (k_sc2_mma: cb >= rb*128 // TN), K = 32W
            tn = 240 if MMA_FP4 else 256
            cbs = -(-h // tn)
            tiles = sum(cbs - rb * 128 // tn for rb in range(-(-h // 128)))
            mma_ops += tiles * 2 * 128 * tn * 32 * W
            mma_useful += h * (h - 1) // 2 * 2 * 32 * W  # the upper H x H pairs the method needs, K = N rounded to 32
            hp = max(-(-h // 256) * 256, -(-h // 240) * 240 + 16)
            expand_bytes += hp * 16 * W + h * (4 * W + 8 * W)  # X rows (e2m1) written, rows read, UP written
    score_tests = int(sum(int(r["hypotheses_evaluated"]) for r in res)) * CFG.n
    return {"compat_tests": tests, "mma_ops": mma_ops, "mma_useful_ops": mma_useful, "score_tests": score_tests,
            "edges": edges,
            "degree_bytes": deg_bytes, "expand_bytes": expand_bytes}


# instructions per 64 tests (one warp instruction = 32 lanes x 2 packed tests) that occupy the FP32 pipe:
# packed FP (FFMA2/FADD2/FMUL2) and 32-bit integer ALU ops, which tools/fp32_pipe_probe.cu shows cost the
# same pipe time as an FFMA2 on this part; each takes 2 cycles of a sub-partition's pipe
ISSUE_MIX = {"k_compat": (19, 8), "k_score": (16, 2)}


def rooflines(kern, work, steps, pk, pairs):
    """Per-kernel roofline entries (achieved algorithmic rate ÷ peak) from CUDA-event kernel times, for every
    kernel with a defined bound; ncu-derived fields (traffic, IPC, L2 hit rate) from the committed summary."""
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    fp32_peak = SMS * 128 * sm_max * 1e6 / 1e12  # T lane-ops/s, one fp32 op per lane per clock
    hbm_peak = float(pk.get("hbm_gbs", 6650.0)) / 1000.0  # TB/s
    # dense-block peak from the measured bf16 figure x the guide's nominal ratio: fp4 9/2.25, int8 4.5/2.25
    mma_peak = (4.0 if MMA_FP4 else 2.0) * float(pk.get("bf16_tflops", 1590.0))
    out = {}

    def entry(name, bound, units, peak, unit, per_unit, tests=None):
        ms, launches = kern.get(name, (0.0, 0))
        if not launches or not ms:
            return
        t = ms / launches / 1000.0
        e = {"bound": bound, "measured_ms_per_launch": t * 1000, "per_unit": per_unit}
        if units is not None:
            ach = units / t / 1e12
            e.update(achieved=ach, peak=peak, unit=unit, frac=ach / peak)
        tr = ncu_traffic(name)
        e["traffic"] = (tr["dram_bytes_per_pair"] * pairs) if tr else None
        e["traffic_source"] = (tr["source"] + " (ncu --set full dram read+write per pair x pairs)") if tr else None
        nc = ncu_metrics(name)
        if nc:
            e["ncu"] = {k: round(v, 3) for k, v in nc.items() if k in ("ipc", "l2_hit_pct", "dram_pct", "fma_pipe_pct",
                                                                          "alu_pipe_pct", "tensor_pipe_pct", "occupancy_pct")}
            if units is None:  # issue-bound kernels: warp instructions issued per cycle per SM, of 4
                e.update(achieved=nc.get("ipc", 0.0), peak=4.0, unit="warp-instr/clk/SM (ncu)",
                         frac=nc.get("ipc", 0.0) / 4.0)
        if name in ISSUE_MIX and tests:
            fp, alu = ISSUE_MIX[name]
            t_issue = (fp + alu) * 2.0 * tests / 64.0 / (4 * SMS * sm_max * 1e6)
            e["issue_bound"] = {"fp2_plus_alu_instr_per_64_tests": fp + alu, "bound_ms": t_issue * 1000,
                                "frac": t_issue / t}
        out[name] = e

    entry("k_compat", "alu", work["compat_tests"] * 20, fp32_peak, "T lane-ops/s (fp32)",
          "20 fp32 ops of the Eq. 1 tree per pair test; N(N-1)/2 tests per pair", tests=work["compat_tests"])
    entry("k_score", "alu", work["score_tests"] * 15, fp32_peak, "T lane-ops/s (fp32)",
          "15 FMA-pipe ops of the r13 tree per residual test; hypotheses x N tests per pair",
          tests=work["score_tests"])
    entry("k_sc2_mma", "tensor", work["mma_useful_ops"], mma_peak, "TOPS (fp4 e2m1)" if MMA_FP4 else "TOPS (int8)",
          "2K ops per upper pair of the dense block, |H|(|H|-1)/2 pairs, K = 32W (the executed 128 x %d tiles "
          "do tile_ops_per_useful x that)" % (240 if MMA_FP4 else 256))
    if "k_sc2_mma" in out and work["mma_useful_ops"]:
        out["k_sc2_mma"]["tile_ops_per_useful"] = round(work["mma_ops"] / work["mma_useful_ops"], 3)
    entry("k_degree", "hbm", work["degree_bytes"], hbm_peak, "TB/s", "4W bytes per bit row read + 8 B per row")
    entry("k_expand", "hbm", work["expand_bytes"], hbm_peak, "TB/s",
          "16W B per X row (e2m1) + 12W B per heavy row (row read, UP written)")
    for k in ("k_hist_hi", "k_hist_lo", "k_collect"):
        entry(k, "hbm", work["edges"] * 4, hbm_peak, "TB/s", "4 B per O2 edge per pass")
    for k in ("k_sc2", "k_sc2_light", "k_pgs"):
        entry(k, "issue", None, None, None, "latency/issue-bound list and bitmap intersections (DESIGN.md §6)")
    return out


def ncu_metrics(kernel):
    """ncu --set full metrics of `kernel` from the newest committed profiles/*/ncu_full_summary.json, or None."""
    import glob

    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_full_summary.json")), reverse=True):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        for k, v in d.items():
            if k.split("<")[0].split("(")[0].replace("void ", "").strip() == kernel:
                return v
    return None


# ------------------------------------------------------------------------------------------ host cores / oracle
def host_cores():
    """(usable core count, CPU model line) of this host."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = "unknown"
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


def _oracle_pair(pair):
    """One config-E pair through the oracle (a worker of the all-core pool); returns seconds."""
    import oracle

    inst = synth.workload_instance(CFG, pair=pair)
    t0 = time.perf_counter()
    r = oracle.estimate(inst["src"], inst["dst"], CFG.tau, CFG.k1, CFG.k2, CFG.inlier_threshold)
    dt = time.perf_counter() - t0
    assert r["status"] == 0
    return dt


def _oracle_pool(workers):
    import multiprocessing as mp

    return mp.get_context("spawn").Pool(workers)  # spawn: the parent may hold a CUDA context


def cpu_sample():
    """The oracle as it stands on the host: (i) throughput of a process pool over all usable cores on a
    fixed config-E sample (2 pairs per worker); (ii) single-core latency per config A-D."""
    import oracle

    oracle.build()
    cores, model = host_cores()
    workers = max(1, min(cores, 64))
    npairs = 2 * workers
    with _oracle_pool(workers) as pool:
        pool.map(_oracle_pair, range(10_000, 10_000 + workers))  # warm the workers (import, library load)
        t0 = time.perf_counter()
        per = pool.map(_oracle_pair, range(20_000, 20_000 + npairs), chunksize=1)
        wall = time.perf_counter() - t0
    lat = {}
    for key in "ABCD":
        c = synth.CONFIGS[key]
        inst = synth.workload_instance(c, pair=0)
        reps = 3 if c.n <= 1000 else 1
        ts = []
        for _ in range(reps):
            t1 = time.perf_counter()
            oracle.estimate(inst["src"], inst["dst"], c.tau, c.k1, c.k2, c.inlier_threshold)
            ts.append(time.perf_counter() - t1)
        lat[f"{key} ({c.name}, N={c.n}, K1={c.k1})"] = round(1e3 * float(np.median(ts)), 2)
    return {"value": npairs / wall, "unit": UNIT, "cores": workers, "kind": "oracle",
            "sample": f"{npairs} config-E pairs (N=5000, K1=1000, K2=2, seeds {CFG.seed + 20000}..), a process pool "
                      f"of {workers} single-threaded oracle workers, {wall:.1f} s wall; mean {np.mean(per):.2f} s per "
                      f"pair per core",
            "host": {"usable_cores": cores, "cpu_model": model},
            "single_core_latency_ms": lat}


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The oracle, as it stands, on all usable host cores: each step registers one config-E pair per worker
    (a bounded sample of the workload).  Under torchrun only rank 0 runs it."""
    if rank != 0:
        return
    import oracle

    oracle.build()
    cores, model = host_cores()
    workers = max(1, min(cores, 64))
    times = []
    with _oracle_pool(workers) as pool:
        nxt = 30_000
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_oracle_pair, range(nxt, nxt + workers), chunksize=1)
            dt = time.perf_counter() - t0
            nxt += workers
            if step >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = workers * len(times) / total
    sample = (f"{workers} config-E pairs per step (one per worker), {len(times)} timed steps, process pool of "
              f"{workers} single-threaded C++ oracle workers")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * total / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"configs[4] 3DMatch-shaped pairs (N=5000, K1=1000, K2=2); bounded sample",
                   "pairs_per_step": workers},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "oracle", "sample": sample,
                         "host": {"usable_cores": cores, "cpu_model": model}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ multi-rank plumbing
def _shard(args, rank, world):
    """(first global pair, pairs on this rank, pairs over all ranks, scaling)."""
    from paper_2507_01439_b200.sharding import shard_range

    if args.pairs:
        return rank * args.pairs, args.pairs, world * args.pairs, "weak"
    b, e = shard_range(args.sweep, world, rank)
    return b, e - b, args.sweep, "strong"


def _max_over_ranks(x, world, device):
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_selftest_gloo(args, rank, world):
    """CPU check of the spawn / shard / gather / max-over-ranks path (gloo; no GPU, no method arithmetic):
    every rank fills result records for its shard with values derived from the global pair index, and
    rank 0 checks the gathered array is every pair exactly once in global order."""
    import torch
    import torch.distributed as dist

    from paper_2507_01439_b200._binding import RESULT_DTYPE
    from paper_2507_01439_b200.sharding import gather_results

    first, pairs, total, scaling = _shard(args, rank, world)
    rec = np.zeros(pairs, RESULT_DTYPE)
    rec["inlier_count"] = np.arange(first, first + pairs)
    rec["num_edges"] = 10**9 + np.arange(first, first + pairs)
    dt = _max_over_ranks(1.0 + rank, world, torch.device("cpu"))
    allres = gather_results(rec, total) if world > 1 else rec
    if rank == 0:
        ok = bool((allres["inlier_count"] == np.arange(total)).all() and
                  (allres["num_edges"] == 10**9 + np.arange(total)).all())
        print(json.dumps({"selftest": "gloo", "n_gpus": world, "world": world, "pairs": total, "scaling": scaling,
                          "max_over_ranks": dt, "ok": ok}), flush=True)
    if world > 1:
        dist.barrier()


# ------------------------------------------------------------------------------------------ CUDA arm
def run_cuda(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2507_01439_b200 import RESULT_DTYPE, TurboReg
    from paper_2507_01439_b200._binding import F_KERNEL_TIMING

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    first, pairs, total, scaling = _shard(args, rank, world)
    n = CFG.n
    src_h, dst_h, gts = make_inputs(first, pairs)
    off = (np.arange(pairs) * n).astype(np.int64)
    nn = np.full(pairs, n, np.int32)
    src_d = torch.from_numpy(src_h).to(dev)
    dst_d = torch.from_numpy(dst_h).to(dev)
    out_d = torch.zeros(pairs * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)  # explicit stream: kernels, events and the L2 flush all on it
    torch.cuda.set_stream(stream)
    tr = TurboReg(CFG.tau, CFG.k1, CFG.k2, CFG.inlier_threshold, max_n=n, max_batch=pairs, device=local_rank,
                  max_density=MAX_DENSITY)
    tr.set_option("mma_fp4", MMA_FP4)  # the library default, stated so the roofline below counts the right tiles

    def step():
        tr.register_batch(src_d, dst_d, off, nn, out=out_d, stream=stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    res = out_d.cpu().numpy().view(RESULT_DTYPE).copy()
    if not (res["status"] == 0).all():
        raise RuntimeError(f"rank {rank}: pair statuses {np.unique(res['status'], return_counts=True)}")
    ok = sum(int(synth.rotation_error_deg(r["R"].reshape(3, 3), g[0]) <= 5) for r, g in zip(res, gts))

    # ---- timed region: the default path (CUDA-graph replay + the side stream), device-resident inputs
    clocks = clock_sampler(local_rank)
    clocks.start()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = tr.launch_count
    barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for k in range(args.steps):
        flush.fill_(float(k))  # L2 flush (256 MiB write), outside the event region
        ev0[k].record(stream)
        step()
        ev1[k].record(stream)
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    launches = tr.launch_count - launches0
    clk = clocks.stop()
    dev_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    dev_ms_max = _max_over_ranks(dev_ms, world, dev)
    value = total * args.steps / (dev_ms_max / 1000.0)
    assert out_d.cpu().numpy().view(RESULT_DTYPE).tobytes() == res.tobytes(), "results changed between steps"

    # ---- per-kernel times: a separate pass over the same batch with per-kernel CUDA events (direct launches)
    kp = max(1, min(args.steps, 5))
    tr.set_params(flags=F_KERNEL_TIMING)
    step()
    torch.cuda.synchronize()
    tr.profile_begin()
    for k in range(kp):
        flush.fill_(float(k))
        step()
    torch.cuda.synchronize()
    kern = tr.profile_end()
    tr.set_params(flags=0)
    work = algorithmic_work(tr, res, pairs)

    # ---- end-to-end through the public API with pinned HOST buffers (H2D + D2H inside the timed region)
    src_p = torch.from_numpy(src_h).pin_memory()
    dst_p = torch.from_numpy(dst_h).pin_memory()
    for _ in range(max(1, args.warmup)):
        tr.register_batch(src_p, dst_p, off, nn)
    e2e_times = []
    for k in range(args.steps):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        host_res = tr.register_batch(src_p, dst_p, off, nn)  # blocking: copies in, kernels, result out
        e2e_times.append(time.perf_counter() - t0)
    e2e_value = total * args.steps / _max_over_ranks(sum(e2e_times), world, dev)
    assert host_res.tobytes() == res.tobytes(), "host-input results differ from device-input results"
    ws_bytes = tr.workspace_bytes
    tr.close()

    # gather per-pair results (the only collective: NCCL all_gather of fixed-size records, outside timing)
    if world > 1:
        from paper_2507_01439_b200.sharding import gather_results

        allres = gather_results(res, total)
        all_ok = int((allres["status"] == 0).sum())
    else:
        all_ok = int((res["status"] == 0).sum())

    # context keys never cost the metric line: rank-0-only ones are guarded; the multi-rank split (collectives,
    # where one rank's failure would stall the others) runs only on request
    context = _guarded(single_pair_context, rank, local_rank, stream, src_d, dst_d) \
        if rank == 0 and not args.no_context else None
    split_ctx = split_pair_context(world, local_rank) if world > 1 and args.split_context else None
    split_proj = _guarded(split_phase_projection, local_rank) if world == 1 and not args.no_context else None
    if rank != 0:
        return
    pk = peaks()
    roofs = rooflines(kern, work, kp, pk, pairs)
    # the roofline line describes the dominant kernel (by measured time) among those with a defined bound
    dom_name = max(roofs, key=lambda k: kern[k][0]) if roofs else None
    roof = dict(roofs[dom_name], kernel=dom_name) if dom_name else None
    kms = {k: v[0] / kp for k, v in kern.items() if v[1]}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"configs[4]: {total} 3DMatch-shaped pairs (configs[1] parameters)"
                               + (f", {args.pairs} per GPU" if args.pairs else f", sharded over {world} GPU(s)"),
                   "pairs_total": total, "pairs_rank0": pairs, "N": n, "K1": CFG.k1, "K2": CFG.k2,
                   "tau_m": CFG.tau, "inlier_threshold_m": CFG.inlier_threshold, "inlier_ratio": CFG.inlier_ratio,
                   "l2": "flushed before every timed step (256 MiB write); inputs 24 B x N per pair",
                   "parallelism": f"dp{world} (pairs)", "launch_path": "CUDA graph replay + side stream (default)",
                   "edge_capacity": f"{MAX_DENSITY} of N(N-1)/2 per pair",
                   "workspace_bytes_per_pair": ws_bytes / pairs},
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(src_h.nbytes + dst_h.nbytes),
                "d2h_bytes_per_step": int(pairs * RESULT_DTYPE.itemsize)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "roofline_kernels": roofs,
        "kernels_ms_per_step": kms,
        "kernel_pass": {"what": "per-kernel CUDA events, direct launches on one stream, same batch",
                        "steps": kp, "sum_ms_per_step": sum(kms.values())},
        "planted_recovery": f"{ok}/{pairs} (rank 0, RE<=5deg); all ranks status ok {all_ok}/{total}",
        "wall_s_timed_region": wall,
    }
    line.update(context or {})
    if split_ctx:
        line["split_pair_latency_ms"] = split_ctx
    if split_proj:
        line["split_phase_projection_1gpu"] = {
            "what": "NEXT(1), N = 32768: G logical ranks' phases run one after another on this GPU (projection, "
                    "not a multi-GPU measurement); per phase (compat / SC2 assembly / search) the slowest rank",
            **split_proj}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample()
    print(json.dumps(line), flush=True)


def _median_latency(fn, stream, reps=10, warm=3):
    import torch

    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


def single_pair_context(rank, local_rank, stream, src_d, dst_d):
    """Context numbers (not the metric): single-pair latency of configs A-D and of large N, RANSAC vs TurboReg
    at an equal budget, point-cloud resolution timing."""
    import torch

    from paper_2507_01439_b200 import RESULT_DTYPE, TurboReg

    dev = src_d.device
    o1 = torch.zeros(RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    one = np.zeros(1, np.int64)
    lat_cfg = {}
    for key in "ABCD":
        c = synth.CONFIGS[key]
        inst = synth.workload_instance(c, pair=0)
        nk = inst["src"].shape[0]
        sk, dk = torch.from_numpy(inst["src"]).to(dev), torch.from_numpy(inst["dst"]).to(dev)
        t = TurboReg(c.tau, c.k1, c.k2, c.inlier_threshold, max_n=nk, max_batch=1, device=local_rank)
        nk_ = np.full(1, nk, np.int32)
        lat_cfg[f"{key} ({c.name}, N={nk}, K1={c.k1})"] = _median_latency(
            lambda: t.register_batch(sk, dk, one, nk_, out=o1, stream=stream.cuda_stream), stream)
        t.close()
    # large N (the NEXT(1) question): one 3DMatch-shaped pair per call, configs[1] parameters
    lat_big = {}
    c = synth.CONFIGS["B"]
    for nb in (10_000, 20_000, 32_768):
        inst = synth.workload_instance(c, pair=0, n=nb)
        sk, dk = torch.from_numpy(inst["src"]).to(dev), torch.from_numpy(inst["dst"]).to(dev)
        t = TurboReg(c.tau, c.k1, c.k2, c.inlier_threshold, max_n=nb, max_batch=1, device=local_rank)
        nk_ = np.full(1, nb, np.int32)
        ms = _median_latency(lambda: t.register_batch(sk, dk, one, nk_, out=o1, stream=stream.cuda_stream), stream,
                             reps=5, warm=2)
        r = o1.cpu().numpy().view(RESULT_DTYPE)[0]
        lat_big[f"N={nb}"] = {"ms": ms, "status": int(r["status"]), "edges": int(r["num_edges"]),
                              "recovered": bool(synth.rotation_error_deg(r["R"].reshape(3, 3), inst["R"]) <= 5)}
        t.close()
    # NEXT(4): equal-budget 3-point RANSAC (K1*K2 sampled triples) vs TurboReg on config-C pairs (5 % inliers),
    # host inputs, wall-clock per call; not part of the timed step
    c = synth.CONFIGS["C"]
    budget = c.k1 * c.k2
    trr = TurboReg(c.tau, c.k1, c.k2, c.inlier_threshold, max_n=c.n, max_batch=1, device=local_rank)
    rec_t = rec_r = 0
    inl_t, inl_r, t_t, t_r = [], [], [], []
    npairs = 10
    for q in range(npairs):
        inst = synth.workload_instance(c, pair=500 + q)
        trr.register(inst["src"], inst["dst"])  # warm (graph capture on the first call)
        t0 = time.perf_counter()
        rt = trr.register(inst["src"], inst["dst"])
        t1 = time.perf_counter()
        rr = trr.ransac(inst["src"], inst["dst"], budget, seed=q)
        t2 = time.perf_counter()
        t_t.append(t1 - t0)
        t_r.append(t2 - t1)
        inl_t.append(rt["inlier_count"])
        inl_r.append(rr["inlier_count"])
        rec_t += int(rt["status"] == 0 and synth.rotation_error_deg(rt["R"].reshape(3, 3), inst["R"]) <= 5)
        rec_r += int(rr["status"] == 0 and synth.rotation_error_deg(rr["R"].reshape(3, 3), inst["R"]) <= 5)
    # NEXT(3): point-cloud resolution (tau = 0.25 pr) of device-resident clouds, CUDA-event timed
    res_ms = {}
    for npts in (5000, 32768):
        cloud = torch.from_numpy(
            np.random.default_rng(npts).uniform(-1.5, 1.5, size=(npts, 3)).astype(np.float32)).to(dev)
        trr.point_resolution(cloud)
        ts = []
        for _ in range(5):  # blocking call on the context's own stream: wall clock around it
            t0 = time.perf_counter()
            trr.point_resolution(cloud)
            ts.append(time.perf_counter() - t0)
        res_ms[f"N={npts}"] = round(1e3 * float(np.median(ts)), 4)
    trr.close()
    ransac = {"config": f"C ({c.name}), {npairs} pairs, budget K1*K2 = {budget} hypotheses each",
              "point_resolution_ms": res_ms,
              "turboreg": {"recovered_re_le_5deg": rec_t, "mean_inliers": float(np.mean(inl_t)),
                           "ms_per_pair_host_io": round(1e3 * float(np.median(t_t)), 3)},
              "ransac": {"recovered_re_le_5deg": rec_r, "mean_inliers": float(np.mean(inl_r)),
                         "ms_per_pair_host_io": round(1e3 * float(np.median(t_r)), 3)}}
    return {"single_pair_latency_ms_configs": lat_cfg, "single_pair_latency_ms_large_n": lat_big,
            "ransac_equal_budget": ransac}


def split_pair_context(world, local_rank, n=32768, reps=3):
    """NEXT(1) context (not the metric): one 3DMatch-shaped pair of N = 32768 split over all ranks
    (split.register_split: NCCL all-reduce of C's words and of the edge words, all-gather of the records),
    wall time of the whole call with a barrier on both sides, max over ranks, median of `reps`."""
    import torch
    import torch.distributed as dist

    from paper_2507_01439_b200 import TurboReg
    from paper_2507_01439_b200.split import register_split

    c = synth.CONFIGS["B"]
    inst = synth.workload_instance(c, pair=0, n=n)
    dev = torch.device("cuda", local_rank)
    src, dst = torch.from_numpy(inst["src"]).to(dev), torch.from_numpy(inst["dst"]).to(dev)
    tr = TurboReg(c.tau, c.k1, c.k2, c.inlier_threshold, max_n=n, max_batch=1, device=local_rank, max_density=0.1)
    ts = []
    res = None
    for k in range(reps + 1):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        res = register_split(tr, src, dst)
        torch.cuda.synchronize()
        dist.barrier()
        if k:
            ts.append(_max_over_ranks(time.perf_counter() - t0, world, dev))
    tr.close()
    return {"N": n, "ranks": world, "ms": round(1e3 * float(np.median(ts)), 3), "status": int(res["status"]),
            "inlier_count": int(res["inlier_count"]),
            "recovered": bool(synth.rotation_error_deg(np.asarray(res["R"]).reshape(3, 3), inst["R"]) <= 5)}


def _guarded(fn, *a):
    """A context measurement that must not cost the metric line: its exception becomes an error entry."""
    try:
        return fn(*a)
    except Exception as e:  # noqa: BLE001
        return {"context_error": f"{type(e).__name__}: {e}"[:300]}


def split_phase_projection(local_rank, n=32768, groups=(1, 2, 4), reps=2):
    """NEXT(1) on ONE GPU — a projection, not a multi-GPU measurement: the phases of G logical ranks for one
    N-point pair run one after another on this GPU (the exchanges as device sums, untimed), each rank's
    phase timed with CUDA events on the launching stream; per phase the slowest rank, and their sum, which a
    G-GPU split would take before its exchanges (bytes per rank given; NVLink time not included)."""
    import torch

    from paper_2507_01439_b200 import TurboReg
    from paper_2507_01439_b200._binding import SPLIT_BITS, SPLIT_EDGES, SPLIT_RESULT

    c = synth.CONFIGS["B"]
    inst = synth.workload_instance(c, pair=0, n=n)
    dev = torch.device("cuda", local_rank)
    s = torch.cuda.Stream(device=dev)
    src, dst = torch.from_numpy(inst["src"]).to(dev), torch.from_numpy(inst["dst"]).to(dev)
    out = {}
    for g in groups:
        engines = [TurboReg(c.tau, c.k1, c.k2, c.inlier_threshold, max_n=n, max_batch=1, device=local_rank,
                            max_density=0.1) for _ in range(g)]
        best = None
        for rep in range(reps + 1):
            ph = [[0.0] * g for _ in range(3)]

            def timed(k, r, fn):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                v = fn()
                b.record(s)
                b.synchronize()
                ph[k][r] = a.elapsed_time(b)
                return v

            with torch.cuda.stream(s):
                for r, e in enumerate(engines):
                    timed(0, r, lambda: e.split_begin(src, dst, r, g, stream=s))
                if g > 1:  # each word was written by exactly one rank into zeros: the sum is the all-reduce
                    bits = [e.split_tensor(SPLIT_BITS) for e in engines]
                    tot = sum(b.to(torch.int64) for b in bits).to(torch.int32)
                    for b in bits:
                        b.copy_(tot)
                es = [timed(1, r, lambda: e.split_sc2(stream=s)) for r, e in enumerate(engines)]
                if g > 1 and es[0] > 0:
                    ed = [e.split_tensor(SPLIT_EDGES, es[0]) for e in engines]
                    tot = sum(x.to(torch.int64) for x in ed).to(torch.int32)
                    for x in ed:
                        x.copy_(tot)
                for r, e in enumerate(engines):
                    timed(2, r, lambda: e.split_search(stream=s))
                parts = torch.cat([e.split_tensor(SPLIT_RESULT) for e in engines])
                res = engines[0].split_merge(parts, g, stream=s)
            torch.cuda.synchronize()
            if rep:
                cur = [max(x) for x in ph]
                best = cur if best is None or sum(cur) < sum(best) else best
        E = int(res["num_edges"])
        out[f"G={g}"] = {"phase_ms_max_over_ranks": [round(x, 3) for x in best], "sum_ms": round(sum(best), 3),
                         "exchange_MB_per_rank": round((2 * (g - 1) / g) * (n * ((n + 31) // 32) * 4 + 4 * E) / 1e6, 1),
                         "status": int(res["status"]),
                         "recovered": bool(synth.rotation_error_deg(np.asarray(res["R"]).reshape(3, 3), inst["R"]) <= 5)}
        for e in engines:
            e.close()
    return out


def ncu_traffic(kernel):
    """{dram_bytes_per_pair, source} of `kernel` from the newest committed ncu --set full summary, or None."""
    import glob

    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_traffic.json")), reverse=True):
        try:
            d = json.load(open(f))
            if kernel in d:
                return d[kernel]
        except Exception:
            pass
    return None


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def respawn_under_torchrun(ngpus):
    """`--gpus N` without a torchrun environment: re-launch this command as N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sweep", type=int, default=SWEEP, help="total pairs of the strong-scaling sweep (configs[4])")
    ap.add_argument("--pairs", type=int, default=0, help="weak scaling: this many pairs per GPU instead of --sweep")
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-context", action="store_true", help="skip the single-pair / RANSAC context numbers")
    ap.add_argument("--split-context", action="store_true",
                    help="N > 1: also time one N = 32768 pair split over all ranks (NEXT(1), NCCL exchanges)")
    ap.add_argument("--selftest-gloo", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus < 1 or args.steps < 1 or args.warmup < 0:
        ap.error("bad --gpus/--steps/--warmup")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        respawn_under_torchrun(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    if args.selftest_gloo:
        if world > 1:
            dist.init_process_group("gloo")
        run_selftest_gloo(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return
    if world > 1:
        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, {torch.cuda.device_count()} visible")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines show the rank count
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_cuda(args, rank, world, local_rank)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
