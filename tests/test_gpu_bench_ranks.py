"""The multi-rank bench path (bench.py --gpus N without torchrun: it re-launches
itself through torch.distributed.run) on the one-GPU test box: with
TA_BENCH_SHARE_GPU=1 the two ranks share cuda:0 and reduce over gloo, so the
launcher, shard plan, per-rank engine runs and the max / sum reductions all
execute on a GPU; the driver's N-GPU runs use the same code with NCCL."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
pytestmark = pytest.mark.gpu


def test_two_ranks_share_one_gpu(gpu_engine):
    env = dict(os.environ, TA_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--triplets", "20000", "--no-rows", "--no-affine", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["failed_triplets"] == 0
    assert line["config"]["triplets"] == 20000 and line["config"]["triplets_per_gpu"] == 10000
    assert line["value"] > 0 and line["e2e"]["value"] > 0
