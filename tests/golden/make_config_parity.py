#!/usr/bin/env python3
"""Config-scale parity fixtures, computed BY THE REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libtrioref.so, built from
the unmodified /root/reference sources by oracle/Makefile).  Datasets come from
the reference generator (dataset.cpp:121-211); scores and end coordinates from
the reference batch path run_batch over its tiled engine (dispatch.cpp:119-162,
tiled.cpp:62-71); traceback rows from oracle_align(with_rows)
(oracle.cpp:182-190).  The GPU test tests/test_gpu_config_parity.py compares
the B200 engine with these files bit for bit.

Files (tests/golden/parity/):
  C2_global.npz      all 1,000,000 C2 triplets, global: score (end = (a, b, c))
  C2_sample.npz      every 64th C2 triplet, semi-global + local: score, end
  C2_semi.npz, C2_local.npz   all 1,000,000 C2 triplets, semi-global / local:
                     score (int16) and end (uint8 x 3)
  C3_sample.npz      every 64th C3 triplet (62,500), all three modes
  C4_sample.npz      every 64th C4 triplet (1,563), all three modes
  C5.npz             1000 / 1500 / 2000 bp single triplets, all three modes
  rows_C2.json.gz    first 2,048 C2 triplets x 3 modes: score, end, begin, rows
  rows_C4.json.gz    first 200 of the C4 sample x 3 modes
  rows_C5a.json.gz   the 1000 bp triplet x 3 modes (4 GB reference tensor each)

Usage: python tests/golden/make_config_parity.py [--only NAME ...]
"""
import argparse
import gzip
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import CONFIGS, load_ref, ref_oracle, triplet  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402

OUT = os.path.join(HERE, "parity")
SCHEME = (1, -1, -2)
STRIDE = 64
THREADS = os.cpu_count() or 8


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, file=sys.stderr, flush=True)


def subset(seqs: np.ndarray, offs: np.ndarray, idx: np.ndarray):
    """Triplets idx of (seqs, offs) as a new contiguous (seqs, offs) pair."""
    lo = offs[3 * idx]
    hi = offs[3 * idx + 3]
    lens = np.stack([offs[3 * idx + d + 1] - offs[3 * idx + d] for d in range(3)], axis=1).reshape(-1)
    new_offs = np.zeros(len(lens) + 1, np.int64)
    new_offs[1:] = np.cumsum(lens)
    parts = [seqs[a:b] for a, b in zip(lo, hi)]
    return np.concatenate(parts) if parts else np.zeros(0, np.uint8), new_offs


def ref_batch(R, seqs, offs, mode):
    t0 = time.time()
    score, end, status, wall = R.run_batch(seqs, offs, SCHEME, mode, tile=16, workers=THREADS, strategy=2,
                                           budget=1 << 40)
    assert (status == 0).all(), "reference failed on some triplets"
    log(f"  mode {mode}: {len(score)} triplets in {time.time() - t0:.1f} s")
    return score, end


def gen(R, name):
    spec, mut, indel, seed = CONFIGS[name]
    t0 = time.time()
    seqs, offs = R.generate(spec, mut, indel, seed)
    log(f"{name}: generated {(len(offs) - 1) // 3} triplets in {time.time() - t0:.1f} s")
    return seqs, offs


def sample_modes(R, name, seqs, offs, idx, modes, path):
    s, o = subset(seqs, offs, idx)
    arrs = {"idx": idx.astype(np.int32)}
    for mode in modes:
        score, end = ref_batch(R, s, o, mode)
        arrs[f"score{mode}"] = score
        arrs[f"end{mode}"] = end
    np.savez_compressed(path, **arrs)
    log(f"{name}: wrote {path}")


def rows_fixture(L, name, seqs, offs, idx, path, threads=THREADS):
    pool = ThreadPoolExecutor(max_workers=threads)
    sb = seqs.tobytes()
    out = {"config": name, "spec": CONFIGS[name][0], "scheme": list(SCHEME), "idx": [int(x) for x in idx],
           "modes": {}}
    for mode in (0, 1, 2):
        t0 = time.time()
        out["modes"][str(mode)] = list(pool.map(
            lambda t: ref_oracle(L, triplet(sb, offs, int(t)), SCHEME, mode, budget=1 << 40), idx))
        log(f"  rows {name} mode {mode}: {len(idx)} in {time.time() - t0:.1f} s")
    with gzip.open(path, "wt") as f:
        json.dump(out, f)
    log(f"{name}: wrote {path}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    args = ap.parse_args()
    want = lambda k: args.only is None or k in args.only  # noqa: E731
    os.makedirs(OUT, exist_ok=True)
    R = Reference()
    L = load_ref()

    if want("C4") or want("rows_C4"):
        seqs, offs = gen(R, "C4")
        n = (len(offs) - 1) // 3
        idx = np.arange(0, n, STRIDE)
        if want("C4"):
            sample_modes(R, "C4", seqs, offs, idx, (0, 1, 2), os.path.join(OUT, "C4_sample.npz"))
        if want("rows_C4"):
            rows_fixture(L, "C4", seqs, offs, idx[:200], os.path.join(OUT, "rows_C4.json.gz"), threads=6)

    if want("C5"):
        arrs = {}
        for name in ("C5a", "C5b", "C5c"):
            seqs, offs = gen(R, name)
            jobs = {mode: None for mode in (0, 1, 2)}
            with ThreadPoolExecutor(max_workers=3) as pool:  # one single-threaded tiled run per mode
                futs = {mode: pool.submit(R.run_batch, seqs, offs, SCHEME, mode, 16, 1, 2, False, 1 << 40)
                        for mode in jobs}
                for mode, f in futs.items():
                    score, end, status, wall = f.result()
                    assert status[0] == 0
                    arrs[f"{name}_score{mode}"] = score
                    arrs[f"{name}_end{mode}"] = end
                    log(f"  {name} mode {mode}: score {score[0]} end {end[0].tolist()} ({wall:.1f} s)")
        np.savez_compressed(os.path.join(OUT, "C5.npz"), **arrs)

    if want("rows_C5a"):
        seqs, offs = gen(R, "C5a")
        rows_fixture(L, "C5a", seqs, offs, np.arange(1), os.path.join(OUT, "rows_C5a.json.gz"), threads=1)

    if want("C2") or want("rows_C2") or want("C2_global") or want("C2_full_modes"):
        seqs, offs = gen(R, "C2")
        n = (len(offs) - 1) // 3
        if want("rows_C2"):
            rows_fixture(L, "C2", seqs, offs, np.arange(2048), os.path.join(OUT, "rows_C2.json.gz"))
        if want("C2"):
            sample_modes(R, "C2", seqs, offs, np.arange(0, n, STRIDE), (1, 2), os.path.join(OUT, "C2_sample.npz"))
        if want("C2_global"):
            score, end = ref_batch(R, seqs, offs, 0)
            lens = np.diff(offs).reshape(-1, 3)
            assert (end == lens).all()
            assert np.abs(score).max() < 32768
            np.savez_compressed(os.path.join(OUT, "C2_global.npz"), score=score.astype(np.int16))
            log("C2: wrote C2_global.npz")
        if want("C2_full_modes"):
            for mode, fname in ((1, "C2_semi.npz"), (2, "C2_local.npz")):
                score, end = ref_batch(R, seqs, offs, mode)
                assert np.abs(score).max() < 32768 and end.min() >= 0 and end.max() < 256
                np.savez_compressed(os.path.join(OUT, fname), score=score.astype(np.int16), end=end.astype(np.uint8))
                log(f"C2: wrote {fname}")
        del seqs, offs

    if want("C3"):
        seqs, offs = gen(R, "C3")
        n = (len(offs) - 1) // 3
        sample_modes(R, "C3", seqs, offs, np.arange(0, n, STRIDE), (0, 1, 2), os.path.join(OUT, "C3_sample.npz"))


if __name__ == "__main__":
    main()
