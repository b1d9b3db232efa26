"""Multi-process CPU tests of the pair-sharded driver logic (gloo backend, world size 2 and 3): shard ranges
cover every pair exactly once and the result gather returns every rank's records in global pair order."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_01439_b200._binding import RESULT_DTYPE
from paper_2507_01439_b200.sharding import gather_results, shard_range


@pytest.mark.parametrize("P,G", [(1623, 8), (1623, 1), (7, 3), (5, 5), (0, 2), (203, 4)])
def test_shard_ranges_partition_pairs(P, G):
    seen = []
    sizes = []
    for r in range(G):
        b, e = shard_range(P, G, r)
        seen.extend(range(b, e))
        sizes.append(e - b)
    assert seen == list(range(P))
    assert max(sizes) - min(sizes) <= 1


def fake_results(b, e):
    res = np.zeros(e - b, RESULT_DTYPE)
    for k, p in enumerate(range(b, e)):
        res[k]["inlier_count"] = 1000 + p
        res[k]["clique"] = (p, p + 1, p + 2)
        res[k]["R"] = np.eye(3).reshape(9) * (p + 1)
        res[k]["num_edges"] = 10**9 + p
    return res


def _worker(rank, world, port, P, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(P, world, rank)
    out = gather_results(fake_results(b, e), P)
    q.put((rank, out.tobytes()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,P", [(2, 11), (3, 10), (2, 1)])
def test_gather_results_gloo(world, P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = fake_results(0, P).tobytes()
    for rank, blob in got:
        assert blob == want, rank


def test_bench_spawns_ranks_and_gathers_gloo():
    """`bench.py --gpus 2` with no torchrun environment re-launches itself as 2 ranks; the shard / gather /
    max-over-ranks plumbing of the 1623-pair sweep runs on gloo and rank 0 sees every pair once, in order."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest-gloo"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0] == {"selftest": "gloo", "n_gpus": 2, "world": 2, "pairs": 1623, "scaling": "strong",
                        "max_over_ranks": 2.0, "ok": True}


def test_bench_reference_arm_json():
    """`bench.py --impl reference`: the oracle on the host cores prints one JSON line with the same metric,
    unit and direction as the CUDA arm, its cpu_baseline (kind, cores, sample) and an e2e record."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    base = json.load(open(os.path.join(root, "BASELINE.json")))
    assert line["impl"] == "reference" and line["metric"] == base["metric"]
    assert line["unit"] == "registrations/s" and line["higher_is_better"] is True and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
