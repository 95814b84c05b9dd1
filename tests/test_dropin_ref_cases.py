"""The reference's OWN unit-test cases against the drop-in library.

oracle/Makefile `dropin-tests` compiles the reference's doctest files
(proj/tests/test_core.cpp, test_dispatch.cpp, test_metrics.cpp unmodified;
test_tiled.cpp minus the three cases that drive tile internals,
oracle/public_cases.py) against OUR headers (paper_2605_28400_b200/csrc/include)
and links them to libtrioalign.so: a reference caller compiles and passes
unchanged.  Host-only cases run here; the whole suite (align, align_packed,
oracle_align and run_batch on the GPU engine) runs with -m gpu."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_unit_tests")
HOST_ONLY = "|".join([
    "sigma", "sop", "identical residues", "scheme validation", "triplet validation", "mode names",
    "coords order", "plan_partition", "dynamic greedy", "strategy names", "tcups", "homology_pairs",
    "spfp", "packed score bound formula",
])


def binary():
    if os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin-tests"], check=True)
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_unit_tests not built (needs the reference sources)")
    return EXE


def run(env_only=None):
    env = dict(os.environ)
    if env_only:
        env["DOCTEST_ONLY"] = env_only
    p = subprocess.run([binary()], capture_output=True, text=True, timeout=1800, env=env)
    return p.returncode, p.stdout + p.stderr


def test_reference_host_cases_pass_against_dropin():
    rc, out = run(HOST_ONLY)
    assert rc == 0, out[-3000:]
    line = [x for x in out.splitlines() if x.startswith("[doctest-shim]")][-1]
    assert int(line.split("test cases:")[1].split("|")[0]) >= 20, line


@pytest.mark.gpu
def test_reference_cases_pass_against_dropin_on_gpu():
    rc, out = run()
    assert rc == 0, out[-3000:]
    assert "| 0 failed | checks:" in out, out[-2000:]
