"""Wave mode (one long triplet spread over every CTA, wavefront.cuh BLK = 2)
needs all CTAs of a round resident at once: consumers spin on faces other CTAs
publish.  The rounds go through cudaLaunchCooperativeKernel, which guarantees
co-residency or fails loudly.  This test keeps a second stream busy with
another process's-worth of work (a long torch matmul chain) while the engine
runs C5-sized wave alignments on its own stream, in a child process under a
timeout so a hang would fail the test instead of wedging the suite; the
results must still equal the reference's (tests/golden/parity/C5.npz)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
pytestmark = pytest.mark.gpu

CHILD = r"""
import os, sys
sys.path.insert(0, os.environ["TA_ROOT"])
import numpy as np, torch
import paper_2605_28400_b200 as ta
z = np.load(os.path.join(os.environ["TA_ROOT"], "tests", "golden", "parity", "C5.npz"))
busy = torch.cuda.Stream()
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
seqs, offs = ta.generate("fixed:1000:1000:1000:1", 0.025, 0.005, 5)
ok = 0
for rep in range(3):
    with torch.cuda.stream(busy):
        x = a
        for _ in range(40):
            x = (x @ a).clamp_(-1, 1)
    for mode in (0, 1, 2):
        out = ta.align_arrays(seqs, offs, ta.ScoringScheme(1, -1, -2), ta.AlignmentMode(mode),
                              cfg=ta.EngineConfig(cell_budget=1 << 40))
        assert out["status"][0] == 0, out["status"]
        assert out["score"][0] == z[f"C5a_score{mode}"][0], (mode, out["score"][0])
        assert list(out["end"][0]) == list(z[f"C5a_end{mode}"][0]), mode
        ok += 1
torch.cuda.synchronize()
print("ok", ok)
"""


def test_wave_mode_with_a_busy_second_stream(gpu_engine):
    env = dict(os.environ, TA_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.strip().endswith("ok 9"), r.stdout
