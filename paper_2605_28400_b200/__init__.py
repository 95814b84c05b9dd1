"""trioalign-b200: B200-native batched exact 3-way alignment (TrioSeq hot path).

Python mirror of the reference `trioalign` C++ API
(/root/reference/proj/include/trioalign/*.hpp): same names, argument meaning
and error classes, implemented over the C-ABI in include/trioalign_capi.h
(libtrioalign_b200.so, sm_100a kernels).  There is no CPU fallback: calls
that compute alignments raise CudaError when the extension or the GPU is
unavailable.  Pure host-side helpers (plan_partition, packed_score_bound, ...)
work without a GPU.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "ScoringScheme", "make_scheme", "AlignmentMode", "mode_name", "mode_from_name", "Coords",
    "Triplet", "AlignmentResult", "LaneMode", "EngineConfig", "Strategy", "strategy_name",
    "strategy_from_name", "PartitionPlan", "TripletOutcome", "WorkerStats", "BatchReport",
    "align", "align_packed", "oracle_align", "run_batch", "plan_partition", "packed_score_bound",
    "packed_bound_ok", "derive_team_width", "tcups", "align_arrays", "DeviceBatch", "lib",
    "generate", "triplets_from_arrays", "device_count", "last_stats",
    "TrioalignError", "ParseError", "CapacityError", "ConfigError", "ShapeMismatchError",
    "LaneOverflowError", "MalformedAlignmentError", "LogicError", "CudaError", "KGAP",
    "K_ORACLE_CELL_BUDGET", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtrioalign_b200.so")
KGAP = "-"
K_ORACLE_CELL_BUDGET = 1 << 27   # oracle.hpp:12
K_ENGINE_CELL_BUDGET = 1 << 31   # tiled.hpp:26


# ---------------------------------------------------------------------------
# errors (errors.hpp:9-37 + std exceptions)

class TrioalignError(RuntimeError):
    code = 11


class ParseError(TrioalignError):
    code = 1


class CapacityError(TrioalignError):
    code = 2


class ConfigError(TrioalignError):
    code = 3


class ShapeMismatchError(TrioalignError):
    code = 4


class LaneOverflowError(TrioalignError):
    code = 5


class MalformedAlignmentError(TrioalignError):
    code = 6


class InvalidArgument(TrioalignError, ValueError):
    code = 7


class LogicError(TrioalignError):
    code = 8


class CudaError(TrioalignError):
    code = 9


_ERRORS = {c.code: c for c in (ParseError, CapacityError, ConfigError, ShapeMismatchError,
                               LaneOverflowError, MalformedAlignmentError, InvalidArgument,
                               LogicError, CudaError)}


def _raise(code: int, msg: str):
    raise _ERRORS.get(code, TrioalignError)(msg)


# ---------------------------------------------------------------------------
# C-ABI binding

class _Scheme(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32), ("gap", ctypes.c_int32),
                ("gap_open", ctypes.c_int32)]


class _Options(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("with_rows", ctypes.c_int32),
                ("tile_size", ctypes.c_int32), ("team_width", ctypes.c_int32),
                ("team_threads", ctypes.c_int32), ("lane_mode", ctypes.c_int32),
                ("cell_budget", ctypes.c_uint64), ("gap_model", ctypes.c_int32)]


class _Results(ctypes.Structure):
    _fields_ = [("scores", ctypes.c_void_p), ("ends", ctypes.c_void_p),
                ("begins", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("rows0", ctypes.c_void_p), ("rows1", ctypes.c_void_p),
                ("rows2", ctypes.c_void_p), ("row_offsets", ctypes.c_void_p),
                ("row_lens", ctypes.c_void_p)]


class _Stats(ctypes.Structure):
    _fields_ = [("kernel_ms", ctypes.c_double), ("wavefront_ms", ctypes.c_double),
                ("cells", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("padded_cells", ctypes.c_int64), ("lanes", ctypes.c_int32),
                ("buckets", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("walker_ms", ctypes.c_double), ("dir_bytes", ctypes.c_int64)]


_LIB = None

EXPORTED_SYMBOLS = (
    "ta_last_error", "ta_version", "ta_device_count", "ta_align_batch", "ta_batch_create",
    "ta_batch_run", "ta_batch_fetch", "ta_batch_stats", "ta_last_stats", "ta_batch_destroy",
    "ta_packed_score_bound", "ta_derive_team_width", "ta_validate_scheme",
    "ta_validate_options", "ta_plan_partition", "ta_generate", "ta_generate_slice", "ta_generate_reference",
    "ta_generate_error", "ta_free",
)


def lib() -> ctypes.CDLL:
    """Loads libtrioalign_b200.so (built in-tree by `make -C paper_2605_28400_b200`)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("TA_LIB_PATH_EXPERIMENT", LIB_PATH)  # dev-only: A/B a variant build of the same ABI
    if not os.path.exists(path):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                          "(the B200 engine has no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.ta_last_error.restype = ctypes.c_char_p
    L.ta_version.restype = ctypes.c_char_p
    L.ta_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    L.ta_align_batch.argtypes = [ctypes.c_int, vp, vp, i64, ctypes.POINTER(_Scheme),
                                 ctypes.POINTER(_Options), ctypes.POINTER(_Results), vp]
    L.ta_batch_create.argtypes = [ctypes.c_int, vp, vp, i64, ctypes.POINTER(vp), vp]
    L.ta_batch_run.argtypes = [vp, ctypes.POINTER(_Scheme), ctypes.POINTER(_Options), vp]
    L.ta_batch_fetch.argtypes = [vp, ctypes.POINTER(_Results), vp]
    L.ta_batch_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
    L.ta_last_stats.argtypes = [ctypes.c_int, ctypes.POINTER(_Stats)]
    L.ta_batch_destroy.argtypes = [vp]
    L.ta_batch_destroy.restype = None
    L.ta_packed_score_bound.argtypes = [i64, i64, i64, ctypes.POINTER(_Scheme)]
    L.ta_packed_score_bound.restype = i64
    L.ta_derive_team_width.argtypes = [i32, i32, i32]
    L.ta_derive_team_width.restype = i32
    L.ta_validate_scheme.argtypes = [ctypes.POINTER(_Scheme)]
    L.ta_validate_options.argtypes = [ctypes.POINTER(_Options)]
    L.ta_plan_partition.argtypes = [vp, i64, i32, i32, vp]
    L.ta_generate.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_double, u64, ctypes.c_int,
                              ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.ta_generate_slice.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_double, u64, i64, i64,
                                    ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.ta_generate_reference.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_double, u64,
                                        ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                        ctypes.POINTER(i64)]
    L.ta_generate_error.restype = ctypes.c_char_p
    L.ta_free.argtypes = [vp]
    L.ta_free.restype = None
    _LIB = L
    return L


def _check(rc: int):
    if rc != 0:
        _raise(rc, lib().ta_last_error().decode(errors="replace"))


def last_stats(device: int = 0) -> dict:
    """Engine statistics of the last one-shot call (ta_align_batch) on a device."""
    st = _Stats()
    _check(lib().ta_last_stats(device, ctypes.byref(st)))
    return {k: getattr(st, k) for k, _ in _Stats._fields_}


def device_count() -> int:
    c = ctypes.c_int(0)
    lib().ta_device_count(ctypes.byref(c))
    return c.value


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# domain types (core.hpp)

@dataclass(frozen=True)
class ScoringScheme:
    match: int = 1
    mismatch: int = -1
    gap: int = -2
    gap_open: int = 0  # not in the reference: affine model of SPEC-AFFINE.md (0 = linear)

    def validate(self) -> None:  # core.cpp:10-18
        if self.match <= 0:
            raise InvalidArgument("match score must be positive")
        if self.mismatch > 0:
            raise InvalidArgument("mismatch score must be <= 0")
        if self.gap > 0:
            raise InvalidArgument("gap score must be <= 0")
        if max(abs(self.match), abs(self.mismatch), abs(self.gap)) > 1024:
            raise InvalidArgument("score magnitudes must be <= 1024")
        if self.gap_open > 0:
            raise InvalidArgument("gap open score must be <= 0")
        if abs(self.gap_open) > 1024:
            raise InvalidArgument("score magnitudes must be <= 1024")

    def _c(self) -> _Scheme:
        return _Scheme(self.match, self.mismatch, self.gap, self.gap_open)


def make_scheme(match: int, mismatch: int, gap: int) -> ScoringScheme:
    s = ScoringScheme(match, mismatch, gap)
    s.validate()
    return s


def sigma(x: str, y: str, s: ScoringScheme) -> int:  # core.hpp:36-41
    gx, gy = x == KGAP, y == KGAP
    if gx and gy:
        return 0
    if gx or gy:
        return s.gap
    return s.match if x == y else s.mismatch


def sop(x: str, y: str, z: str, s: ScoringScheme) -> int:  # core.hpp:44-46
    return sigma(x, y, s) + sigma(x, z, s) + sigma(y, z, s)


class AlignmentMode(enum.IntEnum):
    Global = 0
    SemiGlobal = 1
    Local = 2


_MODE_NAMES = {AlignmentMode.Global: "global", AlignmentMode.SemiGlobal: "semiglobal",
               AlignmentMode.Local: "local"}


def mode_name(m: AlignmentMode) -> str:
    return _MODE_NAMES[AlignmentMode(m)]


def mode_from_name(name: str) -> AlignmentMode:  # core.cpp:35-41
    for k, v in _MODE_NAMES.items():
        if v == name:
            return k
    raise ParseError(f"unknown alignment mode '{name}' (expected global, semiglobal, or local)")


Coords = Tuple[int, int, int]


@dataclass
class Triplet:
    id: str
    s0: str
    s1: str
    s2: str

    def cell_count(self) -> int:
        return len(self.s0) * len(self.s1) * len(self.s2)

    def validate(self) -> None:  # core.cpp:43-52
        for seq in (self.s0, self.s1, self.s2):
            for ch in seq:
                if ch not in "ACGT":
                    raise ParseError(f"triplet '{self.id}': invalid character '{ch}' (alphabet is "
                                     "ACGT, gaps are not allowed in inputs)")


@dataclass
class AlignmentResult:
    score: int = 0
    mode: AlignmentMode = AlignmentMode.Global
    end: Coords = (0, 0, 0)
    begin: Coords = (0, 0, 0)
    has_rows: bool = False
    rows: List[str] = field(default_factory=lambda: ["", "", ""])


class LaneMode(enum.IntEnum):
    Single32 = 0
    PackedDual16 = 1


@dataclass
class EngineConfig:  # tiled.hpp:18-30
    tile_size: int = 8
    team_width: int = 0
    lane_mode: LaneMode = LaneMode.Single32
    cell_budget: int = K_ENGINE_CELL_BUDGET
    team_threads: int = 1
    gap_model: int = 0  # 1: force the affine kernels (SPEC-AFFINE.md) even when gap_open == 0

    def validate(self) -> None:  # tiled.cpp:8-15
        if self.tile_size < 1 or self.tile_size > 4096:
            raise ConfigError(f"tile size must be in [1, 4096], got {self.tile_size}")
        if self.team_width < 0:
            raise ConfigError("team width must be >= 0")
        if self.team_threads < 1:
            raise ConfigError("team threads must be >= 1")
        if self.cell_budget == 0:
            raise ConfigError("cell budget must be positive")


def packed_score_bound(t: Triplet, s: ScoringScheme) -> int:  # tiled.cpp:23-29
    chars = len(t.s0) + len(t.s1) + len(t.s2)
    return chars * max(3 * abs(s.match), 3 * abs(s.mismatch), 2 * abs(s.gap))


def packed_bound_ok(t: Triplet, s: ScoringScheme) -> bool:  # tiled.cpp:31-33
    return packed_score_bound(t, s) <= 32767


def derive_team_width(tile_size: int, b: int, c: int) -> int:  # tiled.cpp:17-21
    need = max(b, c)
    if need <= 0:
        return 1
    return (need + tile_size - 1) // tile_size


def tcups(cells: int, seconds: float) -> float:  # metrics.cpp:11-14
    if seconds <= 0:
        raise ValueError("tcups: runtime must be positive")
    return cells / (seconds * 1e12)


# ---------------------------------------------------------------------------
# seeded synthetic datasets (dataset.cpp:87-211, bit-identical, parallel)

def generate(spec: str, mutation: float = 0.0, indel: float = 0.0, seed: int = 0,
             threads: int = 0, begin: int = 0, end: int = -1) -> Tuple[np.ndarray, np.ndarray]:
    """`trioalign generate --spec SPEC --rates M:I --seed S` as arrays:
    (seqs uint8 ASCII, offsets int64 [3n+1]); [begin, end) selects a shard."""
    L = lib()
    s, o, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = L.ta_generate_slice(spec.encode(), float(mutation), float(indel), int(seed), int(begin),
                             int(end), int(threads), ctypes.byref(s), ctypes.byref(o), ctypes.byref(n))
    if rc:
        _raise(rc, L.ta_generate_error().decode())
    try:
        offs = np.ctypeslib.as_array(ctypes.cast(o, ctypes.POINTER(ctypes.c_int64)),
                                     shape=(3 * n.value + 1,)).copy()
        total = int(offs[-1])
        seqs = np.empty(total + 1, np.uint8)
        ctypes.memmove(seqs.ctypes.data, s, total)
        seqs[total] = 0
    finally:
        L.ta_free(s)
        L.ta_free(o)
    return seqs, offs


def triplets_from_arrays(seqs: np.ndarray, offsets: np.ndarray, prefix: str = "t") -> List[Triplet]:
    raw = seqs.tobytes()
    n = (len(offsets) - 1) // 3
    return [Triplet(f"{prefix}{t}", *(raw[offsets[3 * t + d]:offsets[3 * t + d + 1]].decode()
                                        for d in range(3))) for t in range(n)]


# ---------------------------------------------------------------------------
# array-level batch API (the hot path)

def _pack_inputs(triplets: Sequence[Triplet]):
    parts, offs, pos = [], [0], 0
    for t in triplets:
        for s in (t.s0, t.s1, t.s2):
            b = s.encode("ascii")
            parts.append(b)
            pos += len(b)
            offs.append(pos)
    return np.frombuffer(b"".join(parts) + b"\0", dtype=np.uint8), np.asarray(offs, dtype=np.int64)


def _options(mode, with_rows, cfg: Optional[EngineConfig], cell_budget=None) -> _Options:
    cfg = cfg or EngineConfig()
    budget = cfg.cell_budget if cell_budget is None else cell_budget
    return _Options(int(mode), int(bool(with_rows)), cfg.tile_size, cfg.team_width, cfg.team_threads,
                    int(cfg.lane_mode), budget, int(cfg.gap_model))


def align_arrays(seqs: np.ndarray, offsets: np.ndarray, scheme: ScoringScheme,
                 mode: AlignmentMode = AlignmentMode.Global, cfg: Optional[EngineConfig] = None,
                 with_rows: bool = False, cell_budget: Optional[int] = None, device: int = 0,
                 stream: Optional[int] = None, raw_rows: bool = False) -> dict:
    """One batch through ta_align_batch.  seqs: uint8 ASCII, offsets: int64 [3n+1].
    Returns numpy arrays: score, end (n,3), status, and with rows: begin,
    row_len, rows (list of 3-tuples of str) - or, with raw_rows, the three
    uint8 row planes and row_off (triplet t's rows start at row_off[t])."""
    L = lib()
    seqs = np.ascontiguousarray(seqs, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    n = (len(offsets) - 1) // 3
    score = np.zeros(n, np.int32)
    end = np.zeros((n, 3), np.int32)
    status = np.zeros(n, np.int32)
    res = _Results(_ptr(score).value, _ptr(end).value, None, _ptr(status).value)
    out = {"score": score, "end": end, "status": status}
    if with_rows:
        lens = (offsets[3::3] - offsets[0:-1:3])
        caps = offsets[3::3] - offsets[0:-1:3]
        row_off = np.zeros(n, np.int64)
        if n:
            row_off[1:] = np.cumsum(caps)[:-1]
        total = int(caps.sum()) + 1
        r0, r1, r2 = (np.zeros(total, np.uint8) for _ in range(3))
        begin = np.zeros((n, 3), np.int32)
        row_len = np.zeros(n, np.int32)
        res.begins = _ptr(begin).value
        res.rows0, res.rows1, res.rows2 = _ptr(r0).value, _ptr(r1).value, _ptr(r2).value
        res.row_offsets = _ptr(row_off).value
        res.row_lens = _ptr(row_len).value
        del lens
    sch = scheme._c()
    opt = _options(mode, with_rows, cfg, cell_budget)
    _check(L.ta_align_batch(device, _ptr(seqs), _ptr(offsets), n, ctypes.byref(sch),
                            ctypes.byref(opt), ctypes.byref(res), stream))
    if with_rows and raw_rows:
        out.update(begin=begin, row_len=row_len, row_off=row_off, row_planes=(r0, r1, r2))
    elif with_rows:
        rows = []
        for t in range(n):
            o, ln = int(row_off[t]), int(row_len[t])
            rows.append(tuple(bytes(r[o:o + ln]).decode("ascii") for r in (r0, r1, r2)))
        out.update(begin=begin, row_len=row_len, rows=rows)
    return out


class DeviceBatch:
    """Device-resident batch: inputs packed in HBM once, kernels re-run on demand
    (ta_batch_create / ta_batch_run / ta_batch_fetch)."""

    def __init__(self, seqs: np.ndarray, offsets: np.ndarray, device: int = 0,
                 stream: Optional[int] = None):
        L = lib()
        self._seqs = np.ascontiguousarray(seqs, dtype=np.uint8)
        self._off = np.ascontiguousarray(offsets, dtype=np.int64)
        self.n = (len(self._off) - 1) // 3
        self._h = ctypes.c_void_p()
        _check(L.ta_batch_create(device, _ptr(self._seqs), _ptr(self._off), self.n,
                                 ctypes.byref(self._h), stream))

    def run(self, scheme: ScoringScheme, mode=AlignmentMode.Global,
            cfg: Optional[EngineConfig] = None, stream: Optional[int] = None) -> None:
        sch = scheme._c()
        opt = _options(mode, False, cfg)
        _check(lib().ta_batch_run(self._h, ctypes.byref(sch), ctypes.byref(opt), stream))

    def fetch(self, stream: Optional[int] = None) -> dict:
        score = np.zeros(self.n, np.int32)
        end = np.zeros((self.n, 3), np.int32)
        status = np.zeros(self.n, np.int32)
        res = _Results(_ptr(score).value, _ptr(end).value, None, _ptr(status).value)
        _check(lib().ta_batch_fetch(self._h, ctypes.byref(res), stream))
        return {"score": score, "end": end, "status": status}

    def stats(self) -> dict:
        st = _Stats()
        _check(lib().ta_batch_stats(self._h, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in _Stats._fields_}

    def close(self):
        if self._h:
            lib().ta_batch_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# reference-shaped API (tiled.hpp:34-50, oracle.hpp:42-43, dispatch.hpp)

def _error_message(code: int, t: Triplet, cfg: EngineConfig, rows_budget: Optional[int]) -> str:
    if code == CapacityError.code:
        if rows_budget is not None:
            total = (len(t.s0) + 1) * (len(t.s1) + 1) * (len(t.s2) + 1)
            return (f"tensor of {total} cells exceeds the budget of {rows_budget} "
                    f"(triplet '{t.id}')")
        return (f"triplet '{t.id}' has {t.cell_count()} cells, over the budget of "
                f"{cfg.cell_budget}")
    if code == ConfigError.code:
        try:
            cfg.validate()
        except ConfigError as e:
            return str(e)
        n = cfg.tile_size
        w = cfg.team_width or derive_team_width(n, len(t.s1), len(t.s2))
        return (f"tile grid {n}x{w} cannot cover sequence lengths ({len(t.s1)}, {len(t.s2)})")
    if code == ParseError.code:
        return f"triplet '{t.id}': invalid character (alphabet is ACGT, gaps are not allowed in inputs)"
    if code == LogicError.code:
        return f"traceback: no predecessor reproduces a cell value (triplet '{t.id}')"
    return f"triplet '{t.id}': error {code}"


def _align_many(triplets: Sequence[Triplet], scheme: ScoringScheme, mode, cfg: EngineConfig,
                with_rows=False, rows_budget=None, device: int = 0):
    seqs, offs = _pack_inputs(triplets)
    return align_arrays(seqs, offs, scheme, mode, cfg, with_rows=with_rows,
                        cell_budget=rows_budget, device=device)


def align(t: Triplet, scheme: ScoringScheme, mode: AlignmentMode, cfg: EngineConfig) -> AlignmentResult:
    """tiled.hpp:34-35 — score + end coordinates (no rows)."""
    cfg.validate()
    out = _align_many([t], scheme, mode, cfg)
    code = int(out["status"][0])
    if code:
        _raise(code, _error_message(code, t, cfg, None))
    return AlignmentResult(int(out["score"][0]), AlignmentMode(mode), tuple(int(x) for x in out["end"][0]))


def align_packed(t1: Triplet, t2: Triplet, scheme: ScoringScheme, mode: AlignmentMode,
                 cfg: EngineConfig) -> Tuple[AlignmentResult, AlignmentResult]:
    """tiled.hpp:38-41 — two same-shape triplets; identical results to two
    align() calls (the GPU always packs lanes when the bound is provable)."""
    if (len(t1.s0), len(t1.s1), len(t1.s2)) != (len(t2.s0), len(t2.s1), len(t2.s2)):
        raise ShapeMismatchError(f"packed alignment requires identical sequence lengths "
                                 f"('{t1.id}' vs '{t2.id}')")
    bound = packed_score_bound(t1, scheme)
    if bound > 32767:
        raise LaneOverflowError(f"score bound {bound} does not fit a signed 16-bit lane")
    cfg.validate()
    out = _align_many([t1, t2], scheme, mode, cfg)
    res = []
    for x, t in enumerate((t1, t2)):
        code = int(out["status"][x])
        if code:
            _raise(code, _error_message(code, t, cfg, None))
        res.append(AlignmentResult(int(out["score"][x]), AlignmentMode(mode),
                                   tuple(int(v) for v in out["end"][x])))
    return res[0], res[1]


def oracle_align(t: Triplet, scheme: ScoringScheme, mode: AlignmentMode, with_rows: bool = False,
                 cell_budget: int = K_ORACLE_CELL_BUDGET) -> AlignmentResult:
    """oracle.hpp:42-43 — score/end (+ begin and gapped rows), computed by the
    GPU direction-cube kernel and walker; same CapacityError budget rule."""
    total = (len(t.s0) + 1) * (len(t.s1) + 1) * (len(t.s2) + 1)
    if total > cell_budget:
        raise CapacityError(f"tensor of {total} cells exceeds the budget of {cell_budget} "
                            f"(triplet '{t.id}')")
    out = _align_many([t], scheme, mode, EngineConfig(), with_rows=True, rows_budget=cell_budget)
    code = int(out["status"][0])
    if code:
        _raise(code, _error_message(code, t, EngineConfig(), cell_budget))
    r = AlignmentResult(int(out["score"][0]), AlignmentMode(mode), tuple(int(x) for x in out["end"][0]))
    if with_rows:
        r.begin = tuple(int(x) for x in out["begin"][0])
        r.has_rows = True
        r.rows = list(out["rows"][0])
    return r


class Strategy(enum.IntEnum):
    Blocked = 0
    Interleaved = 1
    Dynamic = 2


def strategy_name(s: Strategy) -> str:
    return ("blocked", "interleaved", "dynamic")[int(s)]


def strategy_from_name(name: str) -> Strategy:
    for s in Strategy:
        if strategy_name(s) == name:
            return s
    raise ParseError(f"unknown partition strategy '{name}' (expected blocked, interleaved, or dynamic)")


@dataclass
class PartitionPlan:
    strategy: Strategy = Strategy.Blocked
    worker_count: int = 1
    assignment: List[int] = field(default_factory=list)


def plan_partition(cell_counts: Sequence[int], strategy: Strategy, worker_count: int) -> PartitionPlan:
    """dispatch.cpp:29-60 (computed by the C-ABI host helper)."""
    L = lib()
    cells = np.ascontiguousarray(cell_counts, dtype=np.uint64)
    out = np.zeros(len(cells), np.int32)
    _check(L.ta_plan_partition(_ptr(cells) if len(cells) else None, len(cells), int(strategy),
                               int(worker_count), _ptr(out) if len(out) else None))
    return PartitionPlan(Strategy(strategy), int(worker_count), [int(x) for x in out])


@dataclass
class TripletOutcome:
    id: str = ""
    worker: int = 0
    cells: int = 0
    ok: bool = False
    score: int = 0
    end: Coords = (0, 0, 0)
    error: str = ""


@dataclass
class WorkerStats:
    assigned: int = 0
    cells: int = 0
    seconds: float = 0.0


@dataclass
class BatchReport:
    per_triplet: List[TripletOutcome] = field(default_factory=list)
    per_worker: List[WorkerStats] = field(default_factory=list)
    wall_seconds: float = 0.0
    scored_cells: int = 0
    tcups: float = 0.0


def run_batch(dataset: Sequence[Triplet], scheme: ScoringScheme, mode: AlignmentMode,
              cfg: EngineConfig, plan: PartitionPlan, devices: Optional[Sequence[int]] = None) -> BatchReport:
    """dispatch.cpp:119-162: workers are GPUs (worker w -> device w mod #devices);
    each worker's triplets go through one batched kernel call; results are
    written back in input order; failures are recorded per triplet."""
    import threading
    import time
    if len(plan.assignment) != len(dataset):
        raise ConfigError(f"partition plan covers {len(plan.assignment)} triplets, dataset has {len(dataset)}")
    W = plan.worker_count
    if any(w < 0 or w >= W for w in plan.assignment):
        raise ConfigError("partition plan names an out-of-range worker")
    rep = BatchReport(per_triplet=[TripletOutcome() for _ in dataset],
                      per_worker=[WorkerStats() for _ in range(W)])
    by_worker: List[List[int]] = [[] for _ in range(W)]
    for i, t in enumerate(dataset):
        w = plan.assignment[i]
        by_worker[w].append(i)
        o = rep.per_triplet[i]
        o.id, o.worker, o.cells = t.id, w, t.cell_count()
        rep.per_worker[w].assigned += 1
        rep.per_worker[w].cells += t.cell_count()
    ndev = max(1, device_count()) if devices is None else len(devices)
    devs = list(devices) if devices is not None else list(range(ndev))
    errors: List[BaseException] = []

    def work(w: int):
        t0 = time.perf_counter()
        idx = by_worker[w]
        if idx:
            try:
                ts = [dataset[i] for i in idx]
                out = _align_many(ts, scheme, mode, cfg, device=devs[w % len(devs)])
                for x, i in enumerate(idx):
                    o = rep.per_triplet[i]
                    code = int(out["status"][x])
                    if code == 0:
                        o.ok, o.score, o.end = True, int(out["score"][x]), tuple(int(v) for v in out["end"][x])
                    else:
                        o.ok, o.error = False, _error_message(code, dataset[i], cfg, None)
            except BaseException as e:  # noqa: BLE001 - recorded, re-raised below
                errors.append(e)
        rep.per_worker[w].seconds = time.perf_counter() - t0

    t0 = time.perf_counter()
    threads = [threading.Thread(target=work, args=(w,)) for w in range(W)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    rep.wall_seconds = time.perf_counter() - t0
    if errors:
        raise errors[0]
    rep.scored_cells = sum(o.cells for o in rep.per_triplet if o.ok)
    rep.tcups = tcups(rep.scored_cells, rep.wall_seconds) if rep.wall_seconds > 0 else 0.0
    return rep
