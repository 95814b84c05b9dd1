"""Multi-rank host logic on CPU (gloo, world_size 2): the bench / run_batch
sharding is the reference's blocked plan (dispatch.cpp:37-41), each rank
generates exactly its own slice of the dataset (per-triplet RNG streams), the
union of the rank-local results equals the single-process result, and the
timing reductions are max / sum over ranks.  The per-triplet compute here is
the CPU oracle (the checker) because this runs without a GPU; on the B200 the
same shards go through the kernels (bench.py)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

SPEC, RATES, SEED = "uniform:0:30:37", (0.05, 0.01), 5


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def worker(rank, world, port, out_q):
    import torch
    import bench
    import paper_2605_28400_b200 as ta
    from oracle.pyoracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = int(SPEC.split(":")[-1])
    lo, hi = bench.shard(n, rank, world)
    seqs, offs = ta.generate(SPEC, *RATES, SEED, begin=lo, end=hi)
    score, end, status = Oracle().batch(seqs, offs, (1, -1, -2), 0)
    cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum()) if hi > lo else 0
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, score.tolist(), end.tolist(), cells))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([float(cells)], dtype=torch.float64)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    if rank == 0:
        out_q.put((gathered, float(t.item()), float(c.item())))
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process():
    import paper_2605_28400_b200 as ta
    from oracle.pyoracle import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax, csum = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = int(SPEC.split(":")[-1])
    # contiguous, disjoint, covering: the blocked plan_partition
    plan = ta.plan_partition([1] * n, ta.Strategy.Blocked, 2).assignment
    spans = [(lo, hi) for lo, hi, *_ in gathered]
    assert spans[0][0] == 0 and spans[0][1] == spans[1][0] and spans[1][1] == n
    for r, (lo, hi) in enumerate(spans):
        assert all(plan[i] == r for i in range(lo, hi))
    seqs, offs = ta.generate(SPEC, *RATES, SEED)
    score, end, _ = Oracle().batch(seqs, offs, (1, -1, -2), 0)
    merged_score = sum((g[2] for g in gathered), [])
    merged_end = sum((g[3] for g in gathered), [])
    assert merged_score == score.tolist()
    assert merged_end == end.tolist()
    assert tmax == 2.0
    assert csum == float(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())


def test_generator_slices_concatenate_to_the_full_dataset():
    import paper_2605_28400_b200 as ta
    seqs, offs = ta.generate(SPEC, *RATES, SEED)
    parts = [ta.generate(SPEC, *RATES, SEED, begin=lo, end=hi) for lo, hi in ((0, 10), (10, 11), (11, 37))]
    cat = b"".join(p[0][:int(p[1][-1])].tobytes() for p in parts)
    assert cat == seqs[:int(offs[-1])].tobytes()


def test_weak_scaling_shards_extend_the_single_gpu_workload():
    """bench.py at N GPUs: N x n triplets of one generator stream, rank r the
    r-th block of n; rank 0's shard is exactly the 1-GPU workload."""
    import bench
    import paper_2605_28400_b200 as ta
    n, world = 12, 3
    one, one_off = ta.generate(f"fixed:20:20:20:{n}", 0.05, 0.01, 2)
    for rank in range(world):
        lo, hi = bench.shard(n * world, rank, world)
        assert (lo, hi) == (rank * n, (rank + 1) * n)
        seqs, offs = ta.generate(f"fixed:20:20:20:{n * world}", 0.05, 0.01, 2, begin=lo, end=hi)
        assert len(offs) == 3 * n + 1
        if rank == 0:
            assert seqs[:int(offs[-1])].tobytes() == one[:int(one_off[-1])].tobytes()


@pytest.mark.parametrize("scaling,total", [("strong", 1000000), ("weak", 2000000)])
def test_bench_launcher_world2(scaling, total):
    """`bench.py --gpus 2` without torchrun re-launches itself through
    torch.distributed.run (2 ranks, 127.0.0.1); --dry-run runs the real
    launcher, shard plan and max / sum reductions on gloo without a GPU."""
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--scaling", scaling], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["total_triplets"] == total and line["covered"] == total and line["max_hi"] == total
    assert line["rank0_shard"] == [0, total // 2] and line["max_rank"] == 1


def test_bench_refuses_missing_gpus():
    """Without enough visible GPUs, --gpus N fails instead of silently
    reporting n_gpus 1."""
    import json
    import subprocess
    import torch
    if torch.cuda.device_count() >= 4:
        pytest.skip("4 GPUs visible")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--no-e2e"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert "GPU(s) visible" in json.loads(r.stdout.strip().splitlines()[-1])["error"]
