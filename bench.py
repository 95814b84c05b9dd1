#!/usr/bin/env python3
"""bench.py — headline benchmark: 3-way GCUPS and triplets/s on the 150 bp batch.

Workload (BASELINE.json configs[1], "C2"): 1,000,000 synthetic triplets from
the reference generator (fixed:150:150:150:1000000, rates 0.025:0.005,
seed 2, bit-identical to /root/reference/proj/src/dataset.cpp), global mode,
scheme {match 1, mismatch -1, gap -2}.  The gap model is LINEAR: the
reference supports only linear gaps, so the affine variant
named in BASELINE.json has no reference to be exact against.
`--workload C3` runs BASELINE's multi-GPU config (4M x 250 bp, seed 3).

  python bench.py [--gpus N --steps K --warmup W]        our engine
  python bench.py --impl reference ...                    reference CPU path

Multi-GPU: one process per GPU.  Under torchrun (WORLD_SIZE set) each rank
takes its GPU; without it, `--gpus N` (N > 1) re-launches itself through
torch.distributed.run with N ranks on 127.0.0.1 (it fails if fewer than N
GPUs are visible).  Scaling ("8 GPUs, same batch"):
  strong (default)  the one batch is split into N contiguous shards
                    (plan_partition "blocked", dispatch.cpp:37-41);
  weak              N x the batch, rank r takes the r-th copy-sized shard.
There is no collective on the data path: barrier + max-reduce of the timings.

A step = one pass of the engine over this rank's shard.
  value  = kernels only, inputs resident in HBM (DeviceBatch), CUDA events on
           the launching stream, L2 flushed (256 MiB write) between steps.
  e2e    = the public API call (ta_align_batch via align_arrays) from host
           ASCII buffers: host 2-bit pack into pinned chunks, H2D, kernels,
           D2H, all inside the timed region (chunks pipelined).
  affine = the same shape through the affine-gap kernels (SPEC-AFFINE.md,
           gap_open -3), kernels only on a 200k-triplet prefix of the shard.
  rows   = score + traceback rows (oracle_align(with_rows) semantics) for C1
           (all 1000 triplets) and a 20k C2 prefix, every mode, through the
           public call from host buffers (e2e) and the engine's own kernel
           time; cpu_baseline = the reference oracle_align on one core.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3-way GCUPS and triplets/s, 150bp batch, 1/2/4/8 B200 vs CPU ref"
WORKLOADS = {
    "C2": {"spec": "fixed:150:150:150:1000000", "rates": (0.025, 0.005), "seed": 2},
    "C3": {"spec": "fixed:250:250:250:4000000", "rates": (0.025, 0.005), "seed": 3},
}
SCHEME = (1, -1, -2)
MODE = 0
OPS_PER_CELL = 13          # 7 add + 6 max per interior cell
INT_LANES_PER_CLK_SM = 64  # measured: VIADDMNMX/VIMNMX3 issue rate (profiles/r01_intpeak.jsonl)
SMS = 148
AFFINE_OPEN = -3           # gap_open of the affine line (SPEC-AFFINE.md)
AFFINE_ALU_PER_CELL = 14   # ALU-pipe instructions per cell-lane of affine.cuh (SASS: VIADDMNMX + VIMNMX3)
AFFINE_OPS_PER_CELL = 39   # SPEC-AFFINE.md "Algorithmic work": algorithmic int ops per affine cell
ROWS_CPU_SAMPLE = 200      # C1 triplets timed through the reference oracle_align (1 core)


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="C2")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong")
    ap.add_argument("--triplets", type=int, default=0, help="override the batch size (debug only)")
    ap.add_argument("--cpu-sample", type=int, default=2048, help="triplets timed on the host CPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-affine", action="store_true")
    ap.add_argument("--no-rows", action="store_true")
    ap.add_argument("--affine-triplets", type=int, default=200000)
    ap.add_argument("--rows-c2", type=int, default=20000, help="C2 prefix of the rows object")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/sharding/reduction path only (no GPU; gloo): prints the rank plan")
    return ap.parse_args(argv)


def workload_spec(args):
    w = WORKLOADS[args.workload]
    spec = w["spec"]
    if args.triplets:
        parts = spec.split(":")
        parts[-1] = str(args.triplets)
        spec = ":".join(parts)
    return spec, int(spec.split(":")[-1])


def shard(n, rank, world):
    chunk = (n + world - 1) // world  # plan_partition blocked
    lo = min(n, rank * chunk)
    return lo, min(n, lo + chunk)


def rank_plan(args, rank, world):
    """(spec of the whole job, lo, hi, total triplets) of this rank's shard."""
    spec, n = workload_spec(args)
    total = n * world if args.scaling == "weak" else n
    parts = spec.split(":")
    parts[-1] = str(total)
    lo, hi = shard(total, rank, world)
    return ":".join(parts), lo, hi, total


# --------------------------------------------------------------------------
# launcher: N ranks on one node without an external torchrun

def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args, argv):
    """If --gpus N > 1 and we are not under torchrun, re-exec through
    torch.distributed.run with N ranks.  Returns an exit code, or None to
    run in this process."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and os.environ.get("TA_BENCH_SHARE_GPU") != "1":
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {have} GPU(s) visible"}))
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


class Dist:
    """Barrier / max / sum over ranks (nccl on GPUs; gloo for --dry-run)."""

    def __init__(self, world, local, backend):
        self.world = world
        self.dist = None
        self.device = None
        if world > 1:
            import torch
            import torch.distributed as dist
            self.dist = dist
            if backend == "nccl":
                self.device = torch.device("cuda", local)
                dist.init_process_group("nccl", device_id=self.device)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def _reduce(self, x, op):
        if not self.dist:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device or "cpu")
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX) if self.dist else x

    def sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM) if self.dist else x

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# --------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None
        self.active = False
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            if self.active:
                self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(s[1]) for s in self.samples if len(s) >= 9 and s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if len(s) >= 9 and s[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples if len(s) >= 9 for i in range(4)
                          if s[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------
# CPU baselines: the reference's own code on the host cores

def cpu_baseline(seqs, offs, sample, scheme, mode):
    n = min(sample, (len(offs) - 1) // 3)
    s_off = offs[:3 * n + 1]
    s_seq = seqs[:int(s_off[-1])]
    cells = int(np.prod(np.diff(s_off).reshape(-1, 3).astype(np.int64), axis=1).sum())
    threads = os.cpu_count() or 1
    try:
        from oracle.pyoracle import Reference
        ref = Reference()
        score, end, status, wall = ref.run_batch(s_seq, s_off, scheme, mode, tile=16, workers=threads,
                                                 strategy=2)
        kind = "reference"
        desc = f"reference run_batch (tiled engine, tile 16, dynamic partition, {threads} workers)"
    except (OSError, FileNotFoundError, RuntimeError):
        from oracle.pyoracle import Oracle
        o = Oracle()
        t0 = time.perf_counter()
        score, end, status = o.batch(s_seq, s_off, scheme, mode, threads=threads)
        wall = time.perf_counter() - t0
        kind = "port"
        desc = f"oracle port (full-tensor fill, {threads} threads)"
    return {"value": cells / wall / 1e9, "unit": "GCUPS", "cores": threads, "kind": kind,
            "sample": f"first {n} triplets of the workload, {desc}", "seconds": wall,
            "triplets_per_s": n / wall, "cells": cells}, (score, end)


def rows_cpu_baseline(seqs, offs, sample):
    """The reference `trioalign oracle` path (oracle_align with rows, single-
    threaded by construction, cli.cpp:166-196) on the first `sample` C1
    triplets, global mode; returns (baseline dict, results for parity)."""
    from oracle.pyoracle import Reference
    ref = Reference()
    n = min(sample, (len(offs) - 1) // 3)
    sb = seqs.tobytes()
    trips = [[sb[offs[3 * t + d]:offs[3 * t + d + 1]].decode() for d in range(3)] for t in range(n)]
    cells = sum(len(t[0]) * len(t[1]) * len(t[2]) for t in trips)
    t0 = time.perf_counter()
    res = [ref.oracle_align(t, SCHEME, 0, with_rows=True) for t in trips]
    wall = time.perf_counter() - t0
    return {"value": cells / wall / 1e9, "unit": "GCUPS", "cores": 1, "kind": "reference",
            "sample": f"first {n} C1 triplets, global, reference oracle_align(with_rows) on 1 core",
            "triplets_per_s": n / wall}, res


# --------------------------------------------------------------------------

def run_reference_arm(args):
    """--impl reference: the reference CPU path timed on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    spec, n_total = workload_spec(args)
    w = WORKLOADS[args.workload]
    sample = min(args.cpu_sample, n_total)
    # the reference's own generate_dataset (dataset.cpp:121-211) on a prefix
    # spec: per-triplet RNG streams make it identical to the first `sample`
    # triplets of the full workload; nothing of ours runs on this arm
    parts = spec.split(":")
    parts[-1] = str(sample)
    try:
        from oracle.pyoracle import Reference
        seqs, offs = Reference().generate(":".join(parts), *w["rates"], w["seed"])
    except (OSError, FileNotFoundError):
        from oracle.pyoracle import Oracle
        seqs, offs = Oracle().generate(":".join(parts), *w["rates"], w["seed"])
    times, cells, last = [], 0, None
    for step in range(args.warmup + args.steps):
        res, _ = cpu_baseline(seqs, offs, sample, SCHEME, MODE)
        if step >= args.warmup:
            times.append(res["seconds"])
            cells = res["cells"]
            last = res
    total = sum(times)
    value = cells * len(times) / total / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GCUPS", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: reference generator, bit-identical inputs",
        "config": {"workload": f"{args.workload} {spec} rates {w['rates'][0]}:{w['rates'][1]} "
                               f"seed {w['seed']}, global, scheme 1/-1/-2 (linear gap); "
                               f"each step times a {sample}-triplet prefix on the host CPU",
                   "triplets_per_step": sample, "cells_per_step": cells},
        "triplets_per_s": sample * len(times) / total,
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def dry_run(args):
    """Launcher + sharding + reduction path without a GPU (gloo): every rank
    reports its shard; rank 0 prints the plan and the reduced totals."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    d = Dist(world, 0, "gloo")
    spec, lo, hi, total = rank_plan(args, rank, world)
    d.barrier()
    covered = d.sum(hi - lo)
    last_hi = d.max(hi)
    slowest = d.max(float(rank))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": args.scaling, "spec": spec,
                          "total_triplets": total, "rank0_shard": [lo, hi], "covered": int(covered),
                          "max_hi": int(last_hi), "max_rank": int(slowest)}), flush=True)
    d.close()
    return 0


def measure_rows(ta, local, sh, rows_c2):
    """Score + traceback rows through the public call (host buffers in and
    out), per case and mode: e2e GCUPS (best of 3 wall) and the engine's own
    device time (wavefront + walker) with the direction-record stream rate."""
    cases = [("C1", "fixed:100:100:100:1000", 0.05, 0.0, 1)]
    if rows_c2:
        cases.append(("C2", f"fixed:150:150:150:{rows_c2}", 0.025, 0.005, 2))
    sch = ta.ScoringScheme(*SCHEME)
    out, c1 = [], None
    for name, spec, mut, ind, seed in cases:
        seqs, offs = ta.generate(spec, mut, ind, seed)
        if name == "C1":
            c1 = (seqs, offs)
        n = (len(offs) - 1) // 3
        cells = int(np.prod(np.diff(offs).reshape(-1, 3).astype(np.int64), axis=1).sum())
        for mode in (0, 1, 2):
            ta.align_arrays(seqs, offs, sch, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40,
                            device=local, stream=sh, raw_rows=True)
            best, st, res = 1e9, None, None
            for _ in range(3):
                t0 = time.perf_counter()
                res = ta.align_arrays(seqs, offs, sch, ta.AlignmentMode(mode), with_rows=True, cell_budget=1 << 40,
                                      device=local, stream=sh, raw_rows=True)
                dt = time.perf_counter() - t0
                if dt < best:
                    best, st = dt, ta.last_stats(local)
            rbytes = int(res["row_len"].astype(np.int64).sum()) * 3
            h2d = int(seqs.nbytes + offs.nbytes)
            out.append({
                "case": f"{name} {spec}", "mode": ["global", "semiglobal", "local"][mode], "triplets": n,
                "e2e_gcups": cells / best / 1e9, "e2e_ms": best * 1e3, "kernel_gcups": cells / st["kernel_ms"] / 1e6,
                "kernel_ms": st["kernel_ms"], "walker_ms": st["walker_ms"],
                "dir_bytes": st["dir_bytes"], "dir_gb_s": st["dir_bytes"] / max(st["wavefront_ms"], 1e-9) / 1e6,
                "dir_bytes_per_cell": st["dir_bytes"] / cells, "lanes": st["lanes"],
                "h2d_bytes": h2d, "d2h_bytes": rbytes + n * 32, "failed": int((res["status"] != 0).sum())})
    return out, c1


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference_arm(args)
    rc = maybe_relaunch(args, argv)
    if rc is not None:
        return rc
    if args.dry_run:
        return dry_run(args)

    import torch
    import paper_2605_28400_b200 as ta

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TA_BENCH_SHARE_GPU=1 (test only): ranks share the visible GPUs round robin
    # and reduce over gloo, so the multi-rank path runs on a one-GPU box
    share = os.environ.get("TA_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(1, torch.cuda.device_count())
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but {torch.cuda.device_count()} GPU(s) visible")
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    # host pack threads of the e2e pipeline: the host's cores shared by the ranks
    os.environ.setdefault("TA_HOST_THREADS", str(max(1, (os.cpu_count() or 1) // max(1, local_world))))
    torch.cuda.set_device(local)
    d = Dist(world, local, "gloo" if share else "nccl")

    w = WORKLOADS[args.workload]
    spec_all, lo, hi, total = rank_plan(args, rank, world)
    seqs, offs = ta.generate(spec_all, *w["rates"], w["seed"], begin=lo, end=hi)
    n = (len(offs) - 1) // 3
    lens = np.diff(offs).reshape(-1, 3).astype(np.int64)
    cells = int(np.prod(lens, axis=1).sum())
    scheme = ta.ScoringScheme(*SCHEME)
    mode = ta.AlignmentMode(MODE)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    # ---- device-resident batch: kernels only ----------------------------
    batch = ta.DeviceBatch(seqs, offs, device=local, stream=sh)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > L2
    for _ in range(args.warmup):
        batch.run(scheme, mode, stream=sh)
    torch.cuda.synchronize()
    out = batch.fetch(stream=sh)
    bad = int((out["status"] != 0).sum())

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    d.barrier()
    torch.cuda.synchronize()
    sampler.active = True
    step_ms, wave_ms = [], []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        batch.run(scheme, mode, stream=sh)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        wave_ms.append(batch.stats()["wavefront_ms"])
    torch.cuda.synchronize()
    sampler.active = False
    d.barrier()
    st = batch.stats()
    t_rank = sum(step_ms) / 1e3
    t_max = d.max(t_rank)
    cells_all = d.sum(cells)
    n_all = d.sum(n)
    value = cells_all * args.steps / t_max / 1e9
    trip_s = n_all * args.steps / t_max
    clocks = sampler.summary()
    sampler.stop()

    # ---- e2e through the public API from host buffers ------------------
    e2e = None
    if not args.no_e2e:
        ta.align_arrays(seqs, offs, scheme, mode, device=local, stream=sh)  # warm
        torch.cuda.synchronize()
        d.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = ta.align_arrays(seqs, offs, scheme, mode, device=local, stream=sh)
        torch.cuda.synchronize()
        t_e2e = d.max(time.perf_counter() - t0)
        if not np.array_equal(res["score"], out["score"]):
            raise SystemExit("e2e and device-resident results differ")
        plens = np.diff(offs).astype(np.int64)
        packed = int(((plens + 15) // 16).sum()) * 4      # 2-bit words
        h2d = packed + n * 32 + n * 16 + 2048              # + descriptors + stream items (+ small plan arrays)
        e2e = {"value": cells_all * args.steps / t_e2e / 1e9, "unit": "GCUPS",
               "triplets_per_s": n_all * args.steps / t_e2e,
               "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(n * (4 + 12)),     # score + end (i, j, k)
               "host_input_bytes_per_step": int(seqs.nbytes + offs.nbytes),
               "ms_per_step": 1e3 * t_e2e / args.steps}

    # ---- affine-gap kernels on the same shape (kernels only, prefix) --------
    aff = None
    if not args.no_affine:
        m = min(n, args.affine_triplets)
        a_off = offs[:3 * m + 1]
        a_seq = seqs[:int(a_off[-1])]
        a_cells = int(np.prod(np.diff(a_off).reshape(-1, 3).astype(np.int64), axis=1).sum())
        asch = ta.ScoringScheme(*SCHEME, gap_open=AFFINE_OPEN)
        ab = ta.DeviceBatch(a_seq, a_off, device=local, stream=sh)
        ab.run(asch, mode, stream=sh)
        torch.cuda.synchronize()
        d.barrier()
        a_ms = []
        for _ in range(max(1, args.steps - 1)):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ab.run(asch, mode, stream=sh)
            e1.record(stream)
            e1.synchronize()
            a_ms.append(e0.elapsed_time(e1))
        ast = ab.stats()
        a_out = ab.fetch(stream=sh)
        t_aff = d.max(sum(a_ms) / 1e3)
        a_val = d.sum(a_cells) * len(a_ms) / t_aff / 1e9
        f_a = clocks["sm_mhz"] or 1965.0
        # instruction bound of the current kernel: ALU-pipe instructions per cell-lane (SASS)
        alu_peak_gcups = SMS * INT_LANES_PER_CLK_SM * f_a * 1e6 / AFFINE_ALU_PER_CELL * ast["lanes"] / 1e9
        # algorithmic roofline (SPEC-AFFINE.md §7): ops per cell against the lane-aware int peak
        peak_ops = SMS * INT_LANES_PER_CLK_SM * 2 * f_a * 1e6 * ast["lanes"] / 1e12
        a_achieved = a_val / world * AFFINE_OPS_PER_CELL / 1e3
        aff = {"value": a_val, "unit": "GCUPS", "gap_open": AFFINE_OPEN,
               "workload": f"first {m} triplets of this rank's shard, global, scheme 1/-1/-2/open {AFFINE_OPEN}",
               "triplets_per_s": d.sum(m) * len(a_ms) / t_aff, "lanes": ast["lanes"],
               "failed_triplets": int((a_out["status"] != 0).sum()),
               "alu_bound_gcups": alu_peak_gcups, "alu_frac": a_val / world / alu_peak_gcups,
               "roofline": {"bound": "int32", "ops_per_cell": AFFINE_OPS_PER_CELL, "achieved": a_achieved,
                            "peak": peak_ops, "unit": "TOP/s", "frac": a_achieved / peak_ops},
               "parity": "affine oracle (tests/test_gpu_affine.py); no reference affine exists"}
        ab.close()

    # ---- traceback rows (rank 0, one GPU) -----------------------------------
    rows = None
    if not args.no_rows and rank == 0 and world == 1:
        rcases, c1 = measure_rows(ta, local, sh, args.rows_c2)
        rows = {"cases": rcases, "algorithmic_dir_bytes_per_cell": 0.375,
                "note": "direction records: 3-bit codes per swept cell (algorithmic 0.375 B/cell), stored as "
                        "40 B per 100-cell tile-slice and lane; dir_bytes_per_cell counts swept (padded) cells "
                        "against real cells; e2e = align_arrays(with_rows) from host ASCII to host row planes"}
        if not args.no_cpu_baseline:
            try:
                rcpu, ref = rows_cpu_baseline(*c1, ROWS_CPU_SAMPLE)
                got = ta.align_arrays(c1[0], c1[1], scheme, ta.AlignmentMode(0), with_rows=True,
                                      cell_budget=1 << 40, device=local, stream=sh)
                for x, r in enumerate(ref):
                    mine = {"score": int(got["score"][x]), "end": got["end"][x].tolist(),
                            "begin": got["begin"][x].tolist(), "rows": list(got["rows"][x])}
                    if mine != r:
                        raise SystemExit(f"rows differ from the reference oracle on C1 triplet {x}")
                rcpu["parity_checked_triplets"] = len(ref)
                rows["cpu_baseline"] = rcpu
            except (OSError, FileNotFoundError) as e:
                rows["cpu_baseline"] = {"unavailable": str(e)}

    if rank != 0:
        d.close()
        return 0

    # ---- roofline (dominant kernel = the wavefront) ---------------------
    # lane-aware: with s16x2 lanes one ALU instruction advances two cells
    f_mhz = clocks["sm_mhz"] or 1965.0
    peak_lane = SMS * INT_LANES_PER_CLK_SM * 2 * f_mhz * 1e6 / 1e12        # T int-ops/s on 32-bit lanes
    peak = peak_lane * st["lanes"]
    launch_s = statistics.median(wave_ms) / 1e3
    achieved = cells * OPS_PER_CELL / launch_s / 1e12 if launch_s > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02b_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {
        "bound": "int32", "achieved": achieved, "peak": peak, "unit": "TOP/s",
        "frac": achieved / peak, "traffic": traffic,
        "peak_source": f"measured {INT_LANES_PER_CLK_SM} lane-instr/clk/SM (VIADDMNMX, profiles/r01_intpeak.jsonl) "
                       f"x 2 ops x {SMS} SMs x {f_mhz:.0f} MHz (median SM clock in the timed region) "
                       f"x {st['lanes']} cells per lane-instruction (s16x2)",
        "achieved_gcups_per_launch": cells / launch_s / 1e9 if launch_s > 0 else 0.0,
        "roofline_gcups": peak * 1e3 / OPS_PER_CELL,
        "lanes": st["lanes"],
        "frac_vs_32bit_lane_peak": achieved / peak_lane,
        "padded_cell_frac": cells / st["padded_cells"] if st["padded_cells"] else None,
    }

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu, (ref_score, ref_end) = cpu_baseline(seqs, offs, args.cpu_sample, SCHEME, MODE)
        m = len(ref_score)
        if not (np.array_equal(ref_score, out["score"][:m]) and np.array_equal(ref_end, out["end"][:m])):
            raise SystemExit("GPU results differ from the CPU baseline on the sample")
        cpu.pop("seconds")
        cpu["parity_checked_triplets"] = m

    line = {
        "metric": METRIC, "value": value, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "int16x2" if st["lanes"] == 2 else "int32",
        "data": "synthetic: reference generator (bit-identical), 2-bit packed in HBM",
        "config": {"workload": f"{args.workload} {spec_all} rates {w['rates'][0]}:{w['rates'][1]} "
                               f"seed {w['seed']}, global, scheme 1/-1/-2 (linear gap)",
                   "triplets": total, "triplets_per_gpu": n, "cells": int(cells_all),
                   "parallelism": f"dp{world} (contiguous shards, {args.scaling} scaling)",
                   "l2": "flushed (256 MiB write) between timed steps"},
        "triplets_per_s": trip_s,
        "failed_triplets": bad,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(st["launches"]) * args.steps,
        "clocks": clocks,
        "affine": aff,
        "rows": rows,
    }
    print(json.dumps(line), flush=True)
    d.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
