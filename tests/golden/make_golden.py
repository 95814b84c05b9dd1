#!/usr/bin/env python3
"""Generates the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs in the build container only (needs /root/reference): builds
oracle/_ref/libtrioref.so from the unmodified reference sources
(oracle/Makefile) and records what the reference produces:

  gen_hashes.json     sha256 of generate_dataset output for every config spec
                      (dataset.cpp:121-211) -> pins our generator bit-for-bit
  kat.json            reference-test known answers (test_oracle.cpp, test_tiled.cpp)
  small_rows.json.gz  random triplets (len <= 24, random schemes) x 3 modes:
                      oracle_align(with_rows) score/end/begin/rows + tiled align
  c1_rows.json.gz     config C1 (fixed:100:100:100:1000, 0.05:0, seed 1), all
                      1000 triplets, global: score/end/begin/rows (the
                      reference `trioalign oracle` payload), + semi/local for 100
  configs.json.gz     C2/C3/C4 prefixes and C5: reference tiled `align` scores
                      and end coordinates (global, + semi/local on C2/C4 samples)

Usage: python tests/golden/make_golden.py [--skip-c5]
"""
import argparse
import ctypes
import gzip
import hashlib
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtrioref.so")

CONFIGS = {
    "C1": ("fixed:100:100:100:1000", 0.05, 0.0, 1),
    "C2": ("fixed:150:150:150:1000000", 0.025, 0.005, 2),
    "C3": ("fixed:250:250:250:4000000", 0.025, 0.005, 3),
    "C4": ("uniform:64:512:100000", 0.08, 0.01, 4),
    "C5a": ("fixed:1000:1000:1000:1", 0.025, 0.005, 5),
    "C5b": ("fixed:1500:1500:1500:1", 0.025, 0.005, 5),
    "C5c": ("fixed:2000:2000:2000:1", 0.025, 0.005, 5),
}


def load_ref():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    L = ctypes.CDLL(REF_SO)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.ref_generate.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_double, u64,
                               ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.ref_generate.restype = i64
    L.ref_free.argtypes = [vp]
    L.ref_last_error.restype = ctypes.c_char_p
    L.ref_align.argtypes = [ctypes.c_char_p, i32, ctypes.c_char_p, i32, ctypes.c_char_p, i32,
                            i32, i32, i32, ctypes.c_int, i32, i32, u64, ctypes.POINTER(i32),
                            ctypes.POINTER(i32)]
    L.ref_oracle_align.argtypes = [ctypes.c_char_p, i32, ctypes.c_char_p, i32, ctypes.c_char_p, i32,
                                   i32, i32, i32, ctypes.c_int, ctypes.c_int, u64,
                                   ctypes.POINTER(i32), ctypes.c_char_p, ctypes.c_char_p,
                                   ctypes.c_char_p]
    return L


def generate(L, spec, mut, indel, seed):
    s, o = ctypes.c_void_p(), ctypes.c_void_p()
    n = L.ref_generate(spec.encode(), mut, indel, seed, ctypes.byref(s), ctypes.byref(o))
    if n < 0:
        raise RuntimeError(L.ref_last_error().decode())
    offs = np.ctypeslib.as_array(ctypes.cast(o, ctypes.POINTER(ctypes.c_int64)), shape=(3 * n + 1,)).copy()
    seqs = ctypes.string_at(s, int(offs[-1]))
    L.ref_free(s)
    L.ref_free(o)
    return seqs, offs


def triplet(seqs, offs, t):
    return tuple(seqs[offs[3 * t + d]:offs[3 * t + d + 1]].decode() for d in range(3))


def ref_align(L, t, sch, mode, tile=16, budget=1 << 40):
    score = ctypes.c_int32()
    end = (ctypes.c_int32 * 3)()
    rc = L.ref_align(t[0].encode(), len(t[0]), t[1].encode(), len(t[1]), t[2].encode(), len(t[2]),
                     sch[0], sch[1], sch[2], mode, tile, 1, budget, ctypes.byref(score), end)
    if rc:
        return {"error": rc}
    return {"score": score.value, "end": list(end)}


def ref_oracle(L, t, sch, mode, budget=1 << 34):
    res = (ctypes.c_int32 * 8)()
    cap = len(t[0]) + len(t[1]) + len(t[2]) + 1
    r = [ctypes.create_string_buffer(cap) for _ in range(3)]
    rc = L.ref_oracle_align(t[0].encode(), len(t[0]), t[1].encode(), len(t[1]), t[2].encode(),
                            len(t[2]), sch[0], sch[1], sch[2], mode, 1, budget, res, r[0], r[1], r[2])
    if rc:
        return {"error": rc}
    ln = res[7]
    return {"score": res[0], "end": list(res[1:4]), "begin": list(res[4:7]),
            "rows": [r[d].raw[:ln].decode() for d in range(3)]}


class Rng:
    """CounterRng (rng.hpp:12-43) so the random corpora are reproducible."""
    M = (1 << 64) - 1

    @staticmethod
    def mix(z):
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & Rng.M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & Rng.M
        return z ^ (z >> 31)

    def __init__(self, seed, stream=0):
        self.key = self.mix(seed ^ 0x9e3779b97f4a7c15) ^ self.mix(stream ^ 0xbf58476d1ce4e5b9)
        self.counter = 0

    def next(self):
        self.counter += 1
        return self.mix((self.key + self.counter * 0x9e3779b97f4a7c15) & Rng.M)

    def below(self, n):
        return 0 if n == 0 else (self.next() * n) >> 64

    def base(self):
        return "ACGT"[self.below(4)]


def random_triplet(rng, max_len):
    return tuple("".join(rng.base() for _ in range(rng.below(max_len + 1))) for _ in range(3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c5", action="store_true")
    args = ap.parse_args()
    L = load_ref()
    pool = ThreadPoolExecutor(max_workers=os.cpu_count() or 8)

    # 1. generator hashes
    hashes = {}
    for name, (spec, mut, indel, seed) in CONFIGS.items():
        count = int(spec.split(":")[-1])
        if count > 100000:  # hash a prefix of the huge configs (same per-triplet streams)
            parts = spec.split(":")
            parts[-1] = "20000"
            spec_h = ":".join(parts)
        else:
            spec_h = spec
        seqs, offs = generate(L, spec_h, mut, indel, seed)
        hashes[name] = {"spec": spec_h, "rates": [mut, indel], "seed": seed,
                        "n": int((len(offs) - 1) // 3), "bytes": int(offs[-1]),
                        "sha256_seqs": hashlib.sha256(seqs).hexdigest(),
                        "sha256_offsets": hashlib.sha256(offs.astype("<i8").tobytes()).hexdigest()}
        print("hash", name, hashes[name]["n"], file=sys.stderr)
    for spec, mut, indel, seed in [("uniform:0:12:300", 0.3, 0.1, 7), ("blocked:5,9,20:30", 0.1, 0.05, 8),
                                   ("cycle:3,17,8:31", 0.2, 0.0, 9), ("fixed:4:7:2:5", 0.0, 0.0, 10)]:
        seqs, offs = generate(L, spec, mut, indel, seed)
        hashes[spec] = {"spec": spec, "rates": [mut, indel], "seed": seed, "n": int((len(offs) - 1) // 3),
                        "bytes": int(offs[-1]), "sha256_seqs": hashlib.sha256(seqs).hexdigest(),
                        "sha256_offsets": hashlib.sha256(offs.astype("<i8").tobytes()).hexdigest()}
    with open(os.path.join(HERE, "gen_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1)

    # 2. known answers from the reference tests
    kat = []
    for t, sch, mode in [(("", "", ""), (1, -1, -2), 0), (("", "", ""), (1, -1, -2), 1),
                         (("", "", ""), (1, -1, -2), 2), (("A", "", ""), (1, -1, -2), 0),
                         (("A", "C", "G"), (1, -1, -2), 0), (("ACG", "ACG", "ACG"), (2, -1, -2), 0),
                         (("AAA", "CCC", "GGG"), (1, -1, -2), 2), (("A", "A", "A"), (1, -1, -2), 0),
                         (("ACGT", "AGT", "ACT"), (1, -1, -2), 0), (("AC", "AC", "GC"), (1, -1, -2), 1),
                         (("AC", "AC", "GC"), (1, -1, -2), 0), (("AAA", "CCC", "GGG"), (1, -1, -2), 1)]:
        kat.append({"t": t, "scheme": sch, "mode": mode, "oracle": ref_oracle(L, t, sch, mode),
                    "tiled": ref_align(L, t, sch, mode, tile=2)})
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    # 3. random small corpus, random schemes, all modes, rows
    rng = Rng(20261017, 1)
    cases = []
    for rep in range(240):
        t = random_triplet(rng, 24 if rep % 3 else 9)
        sch = (1 + rng.below(5), -rng.below(6), -rng.below(6))
        if rep % 7 == 0:
            sch = (1 + rng.below(40), -rng.below(60), -rng.below(30))
        cases.append((t, sch))
    jobs = [(t, sch, mode) for t, sch in cases for mode in (0, 1, 2)]
    res = list(pool.map(lambda j: (ref_oracle(L, *j), ref_align(L, *j, tile=4)), jobs))
    small = [{"t": j[0], "scheme": j[1], "mode": j[2], "oracle": r[0], "tiled": r[1]} for j, r in zip(jobs, res)]
    with gzip.open(os.path.join(HERE, "small_rows.json.gz"), "wt") as f:
        json.dump(small, f)

    # 4. C1 with rows (global: all 1000; semi/local: first 100)
    spec, mut, indel, seed = CONFIGS["C1"]
    seqs, offs = generate(L, spec, mut, indel, seed)
    c1 = {"spec": spec, "rates": [mut, indel], "seed": seed, "scheme": [1, -1, -2], "modes": {}}
    for mode, count in ((0, 1000), (1, 100), (2, 100)):
        c1["modes"][str(mode)] = list(pool.map(lambda t: ref_oracle(L, triplet(seqs, offs, t), (1, -1, -2), mode),
                                               range(count)))
        print("C1 mode", mode, file=sys.stderr)
    with gzip.open(os.path.join(HERE, "c1_rows.json.gz"), "wt") as f:
        json.dump(c1, f)

    # 5. config samples through the reference tiled engine (+ rows on a few)
    out = {}
    samples = {"C2": (64, (0, 1, 2), 8), "C3": (16, (0,), 2), "C4": (48, (0, 1, 2), 0)}
    if not args.skip_c5:
        samples.update({"C5a": (1, (0,), 0), "C5b": (1, (0,), 0), "C5c": (1, (0,), 0)})
    for name, (count, modes, nrows) in samples.items():
        spec, mut, indel, seed = CONFIGS[name]
        parts = spec.split(":")
        parts[-1] = str(count)
        spec_s = ":".join(parts)
        seqs, offs = generate(L, spec_s, mut, indel, seed)
        ent = {"spec": spec, "sample_spec": spec_s, "rates": [mut, indel], "seed": seed,
               "scheme": [1, -1, -2], "lengths": np.diff(offs).reshape(-1, 3).tolist(), "modes": {}}
        for mode in modes:
            ent["modes"][str(mode)] = list(pool.map(
                lambda t: ref_align(L, triplet(seqs, offs, t), (1, -1, -2), mode, tile=16), range(count)))
        if nrows:
            ent["rows_global"] = list(pool.map(
                lambda t: ref_oracle(L, triplet(seqs, offs, t), (1, -1, -2), 0), range(nrows)))
        out[name] = ent
        print("config", name, file=sys.stderr)
    with gzip.open(os.path.join(HERE, "configs.json.gz"), "wt") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
