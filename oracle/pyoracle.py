"""ctypes binding of the parity checkers (TEST INFRASTRUCTURE ONLY).

  Oracle     -> oracle/liboracle.so        C restatement (trio_oracle.c)
  Reference  -> oracle/_ref/libtrioref.so  the reference sources themselves

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  The product (paper_2605_28400_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtrioref.so")
REF_SRC = "/root/reference/proj"


class _Scheme(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32), ("gap", ctypes.c_int32)]


class _Result(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("score", "end_i", "end_j", "end_k", "begin_i",
                                               "begin_j", "begin_k", "row_len")]


def build(ref: bool = True) -> None:
    """Builds liboracle.so (always possible: gcc) and, when the reference
    sources are present (build container only), oracle/_ref."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "ref-tests"], check=True)


class Oracle:
    """The C restatement of fill_tensor / optimal_score / traceback."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = ctypes.CDLL(ORACLE_SO)
        i32, i64, u64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        L.to_oracle_align.argtypes = [ctypes.c_char_p, i32, ctypes.c_char_p, i32, ctypes.c_char_p, i32,
                                      _Scheme, ctypes.c_int, u64, ctypes.POINTER(_Result),
                                      ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p]
        L.to_oracle_batch.argtypes = [vp, vp, i64, _Scheme, ctypes.c_int, u64, ctypes.c_int, vp, vp, vp]
        L.to_generate.argtypes = [ctypes.c_int, i32, i32, i32, vp, i32, i32, ctypes.c_double,
                                  ctypes.c_double, u64, vp, i64, vp]
        L.to_generate.restype = i64
        L.to_rng_next.argtypes = [u64, u64, u64]
        L.to_rng_next.restype = u64
        L.to_sigma.argtypes = [ctypes.c_char, ctypes.c_char, _Scheme]
        L.to_sop.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_char, _Scheme]
        L.to_affine_align.argtypes = [ctypes.c_char_p, i32, ctypes.c_char_p, i32, ctypes.c_char_p, i32,
                                      _Scheme, i32, ctypes.c_int, u64, ctypes.POINTER(_Result),
                                      ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p]
        L.to_affine_rescore.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, i32, i32, _Scheme, i32]
        L.to_affine_rescore.restype = i32
        self.L = L

    def affine(self, t: Sequence[str], scheme: Tuple[int, int, int, int], mode: int,
               with_rows: bool = False, budget: int = 1 << 40) -> dict:
        """SPEC-AFFINE.md alignment; scheme = (match, mismatch, gap, gap_open)."""
        s0, s1, s2 = (x.encode() for x in t)
        res = _Result()
        cap = len(s0) + len(s1) + len(s2) + 1
        rows = [ctypes.create_string_buffer(cap) for _ in range(3)] if with_rows else [None] * 3
        rc = self.L.to_affine_align(s0, len(s0), s1, len(s1), s2, len(s2), _Scheme(*scheme[:3]), scheme[3],
                                    mode, budget, ctypes.byref(res), *rows)
        if rc:
            return {"error": rc}
        out = {"score": res.score, "end": [res.end_i, res.end_j, res.end_k]}
        if with_rows:
            out["begin"] = [res.begin_i, res.begin_j, res.begin_k]
            out["rows"] = [rows[d].raw[:res.row_len].decode() for d in range(3)]
        return out

    def affine_rescore(self, rows, lo: int, hi: int, scheme) -> int:
        r = [x.encode() for x in rows]
        return self.L.to_affine_rescore(r[0], r[1], r[2], lo, hi, _Scheme(*scheme[:3]), scheme[3])

    def align(self, t: Sequence[str], scheme: Tuple[int, int, int], mode: int,
              with_rows: bool = False, budget: int = 1 << 40) -> dict:
        s0, s1, s2 = (x.encode() for x in t)
        res = _Result()
        cap = len(s0) + len(s1) + len(s2) + 1
        rows = [ctypes.create_string_buffer(cap) for _ in range(3)] if with_rows else [None] * 3
        rc = self.L.to_oracle_align(s0, len(s0), s1, len(s1), s2, len(s2), _Scheme(*scheme), mode,
                                    budget, ctypes.byref(res), *rows)
        if rc:
            return {"error": rc}
        out = {"score": res.score, "end": [res.end_i, res.end_j, res.end_k]}
        if with_rows:
            out["begin"] = [res.begin_i, res.begin_j, res.begin_k]
            out["rows"] = [rows[d].raw[:res.row_len].decode() for d in range(3)]
        return out

    def batch(self, seqs: np.ndarray, offsets: np.ndarray, scheme, mode: int, threads: int = 1,
              budget: int = 1 << 40):
        n = (len(offsets) - 1) // 3
        score = np.zeros(n, np.int32)
        end = np.zeros((n, 3), np.int32)
        status = np.zeros(n, np.int32)
        seqs = np.ascontiguousarray(seqs, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.int64)
        self.L.to_oracle_batch(seqs.ctypes.data, offsets.ctypes.data, n, _Scheme(*scheme), mode, budget,
                               threads, score.ctypes.data, end.ctypes.data, status.ctypes.data)
        return score, end, status

    def generate(self, spec: str, mutation: float, indel: float, seed: int):
        kind, *rest = spec.split(":")
        lengths = np.zeros(1, np.int32)
        p = [0, 0, 0]
        if kind == "uniform":
            k, p[0], p[1], count = 0, int(rest[0]), int(rest[1]), int(rest[2])
        elif kind == "fixed":
            k = 1
            p = [int(rest[0]), int(rest[1]), int(rest[2])]
            count = int(rest[3]) if len(rest) > 3 else 1
        else:
            k = 2 if kind == "blocked" else 3
            lengths = np.asarray([int(x) for x in rest[0].split(",")], np.int32)
            count = int(rest[1])
        maxlen = max(p + [int(lengths.max())]) if kind != "uniform" else p[1]
        cap = count * 3 * (2 * maxlen + 8) + 16
        seqs = np.zeros(cap, np.uint8)
        offs = np.zeros(3 * count + 1, np.int64)
        total = self.L.to_generate(k, p[0], p[1], p[2], lengths.ctypes.data, len(lengths), count,
                                   mutation, indel, seed, seqs.ctypes.data, cap, offs.ctypes.data)
        if total < 0:
            raise RuntimeError("generator buffer overflow")
        return seqs[:total], offs


class Reference:
    """The reference's own code (oracle/_ref/libtrioref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = ctypes.CDLL(REF_SO)
        i32, i64, u64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        L.ref_run_batch.argtypes = [vp, vp, i64, i32, i32, i32, ctypes.c_int, i32, i32, ctypes.c_int,
                                    ctypes.c_int, u64, vp, vp, vp, ctypes.POINTER(ctypes.c_double)]
        L.ref_generate.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_double, u64,
                                   ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.ref_generate.restype = i64
        L.ref_free.argtypes = [vp]
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_oracle_align.argtypes = [ctypes.c_char_p, i32, ctypes.c_char_p, i32, ctypes.c_char_p, i32,
                                       i32, i32, i32, ctypes.c_int, ctypes.c_int, u64,
                                       ctypes.POINTER(i32), ctypes.c_char_p, ctypes.c_char_p,
                                       ctypes.c_char_p]
        self.L = L

    def run_batch(self, seqs, offsets, scheme, mode: int, tile: int = 16, workers: int = 1,
                  strategy: int = 2, packed: bool = False, budget: int = 1 << 31):
        n = (len(offsets) - 1) // 3
        score = np.zeros(n, np.int32)
        end = np.zeros((n, 3), np.int32)
        status = np.zeros(n, np.int32)
        wall = ctypes.c_double(0)
        seqs = np.ascontiguousarray(seqs, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.int64)
        rc = self.L.ref_run_batch(seqs.ctypes.data, offsets.ctypes.data, n, scheme[0], scheme[1], scheme[2],
                                  mode, tile, workers, strategy, int(packed), budget, score.ctypes.data,
                                  end.ctypes.data, status.ctypes.data, ctypes.byref(wall))
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())
        return score, end, status, wall.value

    def oracle_align(self, t, scheme, mode: int, with_rows: bool = True, budget: int = 1 << 34):
        """The reference oracle_align (oracle.cpp:182-190): score, end, begin, rows."""
        res = (ctypes.c_int32 * 8)()
        cap = len(t[0]) + len(t[1]) + len(t[2]) + 1
        r = [ctypes.create_string_buffer(cap) for _ in range(3)]
        rc = self.L.ref_oracle_align(t[0].encode(), len(t[0]), t[1].encode(), len(t[1]), t[2].encode(), len(t[2]),
                                     scheme[0], scheme[1], scheme[2], mode, int(with_rows), budget, res,
                                     r[0], r[1], r[2])
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())
        return {"score": res[0], "end": list(res[1:4]), "begin": list(res[4:7]),
                "rows": [r[d].raw[:res[7]].decode() for d in range(3)]}

    def generate(self, spec: str, mutation: float, indel: float, seed: int):
        s, o = ctypes.c_void_p(), ctypes.c_void_p()
        n = self.L.ref_generate(spec.encode(), mutation, indel, seed, ctypes.byref(s), ctypes.byref(o))
        if n < 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        offs = np.ctypeslib.as_array(ctypes.cast(o, ctypes.POINTER(ctypes.c_int64)), shape=(3 * n + 1,)).copy()
        # (string_at takes a C int: batches above 2 GiB, e.g. C3, need the array view)
        seqs = np.ctypeslib.as_array(ctypes.cast(s, ctypes.POINTER(ctypes.c_uint8)), shape=(int(offs[-1]),)).copy()
        self.L.ref_free(s)
        self.L.ref_free(o)
        return seqs, offs
