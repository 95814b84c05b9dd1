"""CLI drop-in parity: our `trioalign` (paper_2605_28400_b200/trioalign, GPU
engine) against the reference's own CLI built unmodified into
oracle/_ref/trioalign_ref (proj/src/cli.cpp + a CLI11 subset shim).  Output
files are compared byte for byte."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OURS = os.path.join(ROOT, "paper_2605_28400_b200", "trioalign")
REF = os.path.join(ROOT, "oracle", "_ref", "trioalign_ref")


def need_ref():
    if not os.path.exists(REF):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        else:
            pytest.skip("oracle/_ref/trioalign_ref not built")


def run(exe, args, cwd):
    return subprocess.run([exe] + args, cwd=cwd, capture_output=True, text=True, timeout=900)


def both(args, tmp_path, outs):
    need_ref()
    res = {}
    for name, exe in (("ref", REF), ("ours", OURS)):
        d = tmp_path / name
        d.mkdir(exist_ok=True)
        for f in os.listdir(tmp_path):
            src = tmp_path / f
            if src.is_file():
                (d / f).write_bytes(src.read_bytes())
        p = run(exe, args, d)
        res[name] = (p.returncode, {o: (d / o).read_bytes() if (d / o).exists() else None for o in outs}, p.stderr)
    return res


SPECS = [("fixed:30:30:30:40", "0.05:0.01", "1"), ("uniform:0:60:50", "0.1:0.02", "7"),
         ("blocked:3,40,17:20", "0.2:0.05", "2"), ("fixed:5:9:2:4", "0:0", "3")]


@pytest.mark.parametrize("spec,rates,seed", SPECS)
def test_generate_identical(tmp_path, spec, rates, seed):
    res = both(["generate", "--spec", spec, "--rates", rates, "--seed", seed, "--out", "d.fa"], tmp_path, ["d.fa"])
    assert res["ref"][0] == res["ours"][0] == 0
    assert res["ref"][1] == res["ours"][1]


def test_usage_errors_same_exit_codes(tmp_path):
    need_ref()
    for args in ([], ["nope"], ["align"], ["generate", "--spec", "bogus:1"], ["align", "--in", "missing.fa"],
                 ["generate", "--spec", "fixed:4:5:6:2", "--ref-out", "r.fa"]):
        a = run(REF, args, tmp_path).returncode
        b = run(OURS, args, tmp_path).returncode
        assert a == b, (args, a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("spec,rates,seed", SPECS)
@pytest.mark.parametrize("mode", ["global", "semiglobal", "local"])
def test_align_oracle_bench_identical(tmp_path, spec, rates, seed, mode):
    need_ref()
    g = run(OURS, ["generate", "--spec", spec, "--rates", rates, "--seed", seed, "--out", "d.fa"], tmp_path)
    assert g.returncode == 0
    common = ["--in", "d.fa", "--mode", mode]
    r = both(["align"] + common + ["--out", "a.csv", "--tile-size", "4", "--workers", "2"], tmp_path, ["a.csv"])
    assert r["ref"][0] == r["ours"][0] == 0
    assert r["ref"][1] == r["ours"][1]
    r = both(["oracle"] + common + ["--out", "o.csv", "--rows-out", "rows.fa"], tmp_path, ["o.csv", "rows.fa"])
    assert r["ref"][0] == r["ours"][0] == 0
    assert r["ref"][1] == r["ours"][1]
    r = both(["bench", "--spec", spec, "--rates", rates, "--seed", seed, "--mode", mode, "--tile-size", "4",
              "--workers", "3", "--partition", "dynamic", "--stable-output", "--out", "b.csv"], tmp_path, ["b.csv"])
    assert r["ref"][0] == r["ours"][0] == 0
    assert r["ref"][1] == r["ours"][1]


@pytest.mark.gpu
def test_cli_capacity_errors_identical(tmp_path):
    need_ref()
    (tmp_path / "big.fa").write_text(">x s0\n" + "ACGT" * 10 + "\n>x s1\n" + "ACGT" * 10 + "\n>x s2\n" + "ACGT" * 10 + "\n")
    r = both(["align", "--in", "big.fa", "--cell-budget", "100", "--tile-size", "4", "--out", "a.csv"], tmp_path, ["a.csv"])
    assert r["ref"][1] == r["ours"][1]
    r = both(["oracle", "--in", "big.fa", "--cell-budget", "100", "--out", "o.csv"], tmp_path, ["o.csv"])
    assert r["ref"][1] == r["ours"][1]


def test_accuracy_identical(tmp_path):
    """`accuracy` (SPFP/SPFN, cli.cpp:227-258, metrics.cpp:16-60) byte for byte:
    estimated = the reference oracle's rows, reference = the generator's true
    alignment; plus the per-alignment 'not the same sequences' row and the
    file-level errors (count mismatch, unequal rows, bad character)."""
    need_ref()
    assert run(REF, ["generate", "--spec", "uniform:0:40:120", "--rates", "0.1:0.05", "--seed", "5", "--out",
                     "d.fa", "--ref-out", "t.fa"], tmp_path).returncode == 0
    assert run(REF, ["oracle", "--in", "d.fa", "--mode", "local", "--rows-out", "e.fa", "--out", "o.csv"],
               tmp_path).returncode == 0
    # a copy of the estimate whose first alignment is over other sequences
    lines = (tmp_path / "e.fa").read_text().splitlines()
    for x, ln in enumerate(lines):
        if not ln.startswith(">") and "A" in ln:
            lines[x] = ln.replace("A", "C", 1)
            break
    (tmp_path / "e2.fa").write_text("\n".join(lines) + "\n")
    (tmp_path / "short.fa").write_text(">a\nAC-\n>b\nA-C\n>c\n--AC\n")
    (tmp_path / "bad.fa").write_text(">a\nAC-\n>b\nANC\n>c\n-AC\n")
    (tmp_path / "two.fa").write_text(">a\nAC\n>b\nAC\n>c\nAC\n" * 2)
    for est, ref in (("e.fa", "t.fa"), ("t.fa", "e.fa"), ("e2.fa", "t.fa"), ("t.fa", "t.fa"),
                     ("two.fa", "t.fa"), ("short.fa", "short.fa"), ("bad.fa", "bad.fa"), ("missing.fa", "t.fa")):
        r = both(["accuracy", "--estimated", est, "--reference", ref, "--out", "acc.csv"], tmp_path, ["acc.csv"])
        assert r["ref"][0] == r["ours"][0], (est, ref, r["ref"][2], r["ours"][2])
        assert r["ref"][1] == r["ours"][1], (est, ref)
        assert r["ref"][2] == r["ours"][2], (est, ref)


def test_fasta_parse_errors_identical_on_large_inputs(tmp_path):
    """The parallel FASTA reader (chunks cut at headers) reports the same
    first error, with the same line number, as the reference's getline
    reader (fasta.cpp:11-68), including through a pipe (`--in -`)."""
    need_ref()
    assert run(REF, ["generate", "--spec", "fixed:150:150:150:60000", "--rates", "0.02:0.01", "--seed", "9",
                     "--out", "d.fa"], tmp_path).returncode == 0
    text = (tmp_path / "d.fa").read_text()
    lines = text.splitlines()
    # a bad residue late in the file and another one later still: the first wins
    for at in (len(lines) * 2 // 3, len(lines) - 5):
        while lines[at].startswith(">"):
            at += 1
        lines[at] = lines[at][:3] + "n" + "X" + lines[at][5:]
    (tmp_path / "bad.fa").write_text("\r\n".join(lines) + "\r\n\n\n")
    (tmp_path / "late_header.fa").write_text(text + ">\nACGT\n")
    (tmp_path / "odd.fa").write_text(text + ">extra\nACGT\n")
    for f in ("bad.fa", "late_header.fa", "odd.fa"):
        r = both(["align", "--in", f, "--out", "a.csv"], tmp_path, [])
        assert r["ref"][0] == r["ours"][0] == 2, (f, r["ref"][2], r["ours"][2])
        assert r["ref"][2] == r["ours"][2], f
    need_ref()
    for exe in (REF, OURS):
        p = subprocess.run(f"cat bad.fa | {exe} align --in - --out a.csv", shell=True, cwd=tmp_path,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 2 and "invalid character 'N'" in p.stderr, (exe, p.stderr)


@pytest.mark.gpu
def test_stdin_pipe_identical(tmp_path):
    """`--in -` from a pipe (not seekable) reaches the engine."""
    need_ref()
    assert run(OURS, ["generate", "--spec", "uniform:0:80:64", "--rates", "0.1:0.02", "--seed", "4", "--out",
                      "d.fa"], tmp_path).returncode == 0
    outs = {}
    for exe in (REF, OURS):
        p = subprocess.run(f"cat d.fa | {exe} align --in - --mode semiglobal", shell=True, cwd=tmp_path,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr
        outs[exe] = p.stdout
    assert outs[REF] == outs[OURS] and outs[OURS].count("\n") == 65
