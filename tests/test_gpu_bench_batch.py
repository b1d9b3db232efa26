"""The exact bench launch (bench.py): the 1623-pair configs[4] sweep as ONE device-resident batch with the
bench's edge capacity, on the default path (CUDA graph + side stream) and on the kernel-timing path; three
pairs (first, middle, last) compared element by element with the oracle (graph, SC², pivots, cliques,
per-hypothesis transforms and counts), 48 more pairs spread over the batch compared on their result records
with the oracle run in a pool of host processes, and both paths bit-identical.  Needs a B200 (≈ 30 GB of
workspace): `pytest -m gpu`."""
import numpy as np
import pytest

import bench
import synth
from tests.gpu_compare import ROT_TOL_RAD, TRANS_TOL, compare_pair

pytestmark = pytest.mark.gpu


def _oracle_record(pair):
    """The oracle's result record for sweep pair `pair` (a worker of a spawn pool)."""
    import oracle

    cfg = bench.CFG
    inst = synth.workload_instance(cfg, pair=pair)
    r = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold)
    keys = ("status", "inlier_count", "clique_weight", "num_pivots", "num_cliques", "hypotheses_evaluated",
            "num_edges")
    return {**{k: int(r[k]) for k in keys}, "clique": tuple(int(x) for x in r["clique"]),
            "R": np.asarray(r["R"], np.float64).reshape(3, 3), "t": np.asarray(r["t"], np.float64)}


def test_bench_batch_against_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01439_b200 import RESULT_DTYPE, TurboReg
    from paper_2507_01439_b200._binding import F_KERNEL_TIMING

    cfg = bench.CFG
    pairs = bench.SWEEP
    src, dst, _ = bench.make_inputs(0, pairs)
    n = cfg.n
    off = (np.arange(pairs) * n).astype(np.int64)
    nn = np.full(pairs, n, np.int32)
    sd, dd = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    out = torch.zeros(pairs * RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n, max_batch=pairs,
                  max_density=bench.MAX_DENSITY)
    for _ in range(2):  # the second call replays the captured graph
        tr.register_batch(sd, dd, off, nn, out=out)
    torch.cuda.synchronize()
    res = out.cpu().numpy().view(RESULT_DTYPE).copy()
    assert (res["status"] == 0).all()
    for p in (0, pairs // 2, pairs - 1):
        r = {k: res[p][k] for k in res.dtype.names}
        compare_pair(tr, p, src[p * n:(p + 1) * n], dst[p * n:(p + 1) * n], cfg.tau, cfg.k1, cfg.k2,
                     cfg.inlier_threshold, result=r)
    # 48 more pairs, every 1623/48-th, on their result records
    import multiprocessing as mp
    import os

    from tests.gpu_compare import rot_angle_rad

    sample = [int(x) for x in np.linspace(1, pairs - 2, 48)]
    workers = max(1, min(len(os.sched_getaffinity(0)), 48))
    with mp.get_context("spawn").Pool(workers) as pool:
        refs = pool.map(_oracle_record, sample)
    for p, ref in zip(sample, refs):
        got = res[p]
        for k in ("status", "inlier_count", "clique_weight", "num_pivots", "num_cliques", "hypotheses_evaluated",
                  "num_edges"):
            assert int(got[k]) == ref[k], (p, k, int(got[k]), ref[k])
        assert tuple(int(x) for x in got["clique"]) == ref["clique"], p
        assert rot_angle_rad(np.asarray(got["R"]).reshape(3, 3), ref["R"]) <= ROT_TOL_RAD, p
        assert np.abs(np.asarray(got["t"], np.float64) - ref["t"]).max() <= TRANS_TOL, p
    tr.set_params(flags=F_KERNEL_TIMING)
    tr.profile_begin()
    tr.register_batch(sd, dd, off, nn, out=out)
    torch.cuda.synchronize()
    prof = tr.profile_end()
    assert prof["k_compat"][1] == 1 and prof["k_score"][1] == 1
    assert out.cpu().numpy().view(RESULT_DTYPE).tobytes() == res.tobytes()
