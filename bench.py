#!/usr/bin/env python3
"""bench.py — headline benchmark: 3-way GCUPS and triplets/s on the 150 bp batch.

Workload (BASELINE.json configs[1], "C2"): 1,000,000 synthetic triplets from
the reference generator (fixed:150:150:150:1000000, rates 0.025:0.005,
seed 2, bit-identical to /root/reference/proj/src/dataset.cpp), global mode,
scheme {match 1, mismatch -1, gap -2}.  The gap model is LINEAR: the
reference supports only linear gaps, so the affine variant
named in BASELINE.json has no reference to be exact against.

  python bench.py [--gpus N --steps K --warmup W]        our engine
  python bench.py --impl reference ...                    reference CPU path

A step = one pass of the engine over this rank's shard of the batch.  With
N GPUs (torchrun, one rank per GPU) the workload is N x 1M triplets of the
same generator stream and rank r takes the contiguous slice [r*1M, (r+1)*1M)
(plan_partition "blocked", dispatch.cpp:37-41) -> weak scaling, per-GPU work
fixed; there is no collective on the data path (barrier + max-reduce of
timings only).

  affine = the same C2 shape through the affine-gap kernels (SPEC-AFFINE.md,
           gap_open -3; the reference has no affine gaps, so this is parity-
           checked against the builder's oracle, not the reference), kernels
           only on a 200k-triplet prefix of this rank's shard.

  value  = kernels only, inputs resident in HBM (DeviceBatch), CUDA events on
           the launching stream, L2 flushed (256 MiB write) between steps.
  e2e    = the public API call (ta_align_batch via align_arrays) from host
           ASCII buffers: host 2-bit pack into pinned chunks, H2D, kernels,
           D2H, all inside the timed region (chunks pipelined).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3-way GCUPS and triplets/s, 150bp batch, 1/2/4/8 B200 vs CPU ref"
WORKLOAD = {
    "name": "C2",
    "spec": "fixed:150:150:150:1000000",
    "rates": (0.025, 0.005),
    "seed": 2,
    "scheme": (1, -1, -2),
    "mode": 0,
}
OPS_PER_CELL = 13          # 7 add + 6 max per interior cell
INT_LANES_PER_CLK_SM = 64  # measured: VIADDMNMX/VIMNMX3 issue rate (profiles/r01_intpeak.jsonl)
SMS = 148
AFFINE_OPEN = -3           # gap_open of the affine line (SPEC-AFFINE.md)


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--triplets", type=int, default=0, help="override the batch size (debug only)")
    ap.add_argument("--cpu-sample", type=int, default=2048, help="triplets timed on the host CPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-affine", action="store_true")
    ap.add_argument("--affine-triplets", type=int, default=200000)
    return ap.parse_args()


def workload_spec(args):
    spec = WORKLOAD["spec"]
    if args.triplets:
        parts = spec.split(":")
        parts[-1] = str(args.triplets)
        spec = ":".join(parts)
    return spec, int(spec.split(":")[-1])


def shard(n, rank, world):
    chunk = (n + world - 1) // world  # plan_partition blocked
    lo = min(n, rank * chunk)
    return lo, min(n, lo + chunk)


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
# CPU baseline: the reference's own run_batch on the host cores

def cpu_baseline(seqs, offs, sample, scheme, mode):
    n = min(sample, (len(offs) - 1) // 3)
    s_off = offs[:3 * n + 1]
    s_seq = seqs[:int(s_off[-1])]
    cells = int(np.prod(np.diff(s_off).reshape(-1, 3).astype(np.int64), axis=1).sum())
    threads = os.cpu_count() or 1
    try:
        from oracle.pyoracle import Reference
        ref = Reference()
        t0 = time.perf_counter()
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


# --------------------------------------------------------------------------

def run_reference_arm(args):
    """--impl reference: the reference CPU path timed on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    spec, n_total = workload_spec(args)
    sample = min(args.cpu_sample, n_total)
    # the reference's own generate_dataset (dataset.cpp:121-211) on a prefix
    # spec: per-triplet RNG streams make it identical to the first `sample`
    # triplets of the full workload; nothing of ours runs on this arm
    parts = spec.split(":")
    parts[-1] = str(sample)
    try:
        from oracle.pyoracle import Reference
        seqs, offs = Reference().generate(":".join(parts), *WORKLOAD["rates"], WORKLOAD["seed"])
    except (OSError, FileNotFoundError):
        from oracle.pyoracle import Oracle
        seqs, offs = Oracle().generate(":".join(parts), *WORKLOAD["rates"], WORKLOAD["seed"])
    times, cells, last = [], 0, None
    for step in range(args.warmup + args.steps):
        res, _ = cpu_baseline(seqs, offs, sample, WORKLOAD["scheme"], WORKLOAD["mode"])
        if step >= args.warmup:
            times.append(res["seconds"])
            cells = res["cells"]
            last = res
    total = sum(times)
    value = cells * len(times) / total / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GCUPS", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic: reference generator, bit-identical inputs",
        "config": {"workload": f"{WORKLOAD['name']} {spec} rates {WORKLOAD['rates'][0]}:{WORKLOAD['rates'][1]} "
                               f"seed {WORKLOAD['seed']}, global, scheme 1/-1/-2 (linear gap); "
                               f"each step times a {sample}-triplet prefix on the host CPU",
                   "triplets_per_step": sample, "cells_per_step": cells},
        "triplets_per_s": sample * len(times) / total,
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import paper_2605_28400_b200 as ta

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    spec, n_total = workload_spec(args)
    # weak scaling: N x n_total triplets of one generator stream, rank r takes the r-th block
    parts = spec.split(":")
    parts[-1] = str(n_total * world)
    spec_all = ":".join(parts)
    lo, hi = shard(n_total * world, rank, world)
    seqs, offs = ta.generate(spec_all, *WORKLOAD["rates"], WORKLOAD["seed"], begin=lo, end=hi)
    n = (len(offs) - 1) // 3
    lens = np.diff(offs).reshape(-1, 3).astype(np.int64)
    cells = int(np.prod(lens, axis=1).sum())
    scheme = ta.ScoringScheme(*WORKLOAD["scheme"])
    mode = ta.AlignmentMode(WORKLOAD["mode"])
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
    st = batch.stats()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    sampler.active = True
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        batch.run(scheme, mode, stream=sh)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    sampler.active = False
    barrier()
    st = batch.stats()
    t_rank = sum(step_ms) / 1e3
    t_max = max_over_ranks(t_rank)
    cells_all = sum_over_ranks(cells)
    n_all = sum_over_ranks(n)
    value = cells_all * args.steps / t_max / 1e9
    trip_s = n_all * args.steps / t_max
    clocks = sampler.summary()
    sampler.stop()

    # ---- e2e through the public API from host buffers ------------------
    e2e = None
    if not args.no_e2e:
        ta.align_arrays(seqs, offs, scheme, mode, device=local, stream=sh)  # warm
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = ta.align_arrays(seqs, offs, scheme, mode, device=local, stream=sh)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0)
        if not np.array_equal(res["score"], out["score"]):
            raise SystemExit("e2e and device-resident results differ")
        lens = np.diff(offs).astype(np.int64)
        packed = int(((lens + 15) // 16).sum()) * 4        # 2-bit words
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
        asch = ta.ScoringScheme(*WORKLOAD["scheme"], gap_open=AFFINE_OPEN)
        ab = ta.DeviceBatch(a_seq, a_off, device=local, stream=sh)
        ab.run(asch, mode, stream=sh)
        torch.cuda.synchronize()
        barrier()
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
        t_aff = max_over_ranks(sum(a_ms) / 1e3)
        a_val = sum_over_ranks(a_cells) * len(a_ms) / t_aff / 1e9
        # affine roofline: 21 ALU-pipe instructions per cell-lane (affine.cuh)
        f_a = 1965.0
        alu_peak_gcups = SMS * INT_LANES_PER_CLK_SM * f_a * 1e6 / 21 * ast["lanes"] / 1e9
        aff = {"value": a_val, "unit": "GCUPS", "gap_open": AFFINE_OPEN,
               "workload": f"first {m} triplets of this rank's shard, global, scheme 1/-1/-2/open {AFFINE_OPEN}",
               "triplets_per_s": sum_over_ranks(m) * len(a_ms) / t_aff, "lanes": ast["lanes"],
               "failed_triplets": int((a_out["status"] != 0).sum()),
               "alu_bound_gcups": alu_peak_gcups, "alu_frac": a_val / world / alu_peak_gcups,
               "parity": "affine oracle (tests/test_gpu_affine.py); no reference affine exists"}
        ab.close()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    # ---- roofline (dominant kernel = the wavefront) ---------------------
    f_mhz = clocks["sm_mhz"] or 1965.0
    peak_int32 = SMS * INT_LANES_PER_CLK_SM * 2 * f_mhz * 1e6 / 1e12   # T int-ops/s (fused instr = 2 ops)
    launch_s = st["wavefront_ms"] / 1e3
    achieved = cells * OPS_PER_CELL / launch_s / 1e12 if launch_s > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {
        "bound": "int32", "achieved": achieved, "peak": peak_int32, "unit": "TOP/s",
        "frac": achieved / peak_int32, "traffic": traffic,
        "peak_source": f"measured {INT_LANES_PER_CLK_SM} lane-instr/clk/SM (VIADDMNMX, profiles/r01_intpeak.jsonl) "
                       f"x 2 ops x {SMS} SMs x {f_mhz:.0f} MHz (median SM clock in the timed region)",
        "achieved_gcups_per_launch": cells / launch_s / 1e9 if launch_s > 0 else 0.0,
        "roofline_gcups": peak_int32 * 1e3 / OPS_PER_CELL,
        "lanes": st["lanes"],
        "lane_peak_frac": achieved / (peak_int32 * st["lanes"]),
        "padded_cell_frac": cells / st["padded_cells"] if st["padded_cells"] else None,
    }

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu, (ref_score, ref_end) = cpu_baseline(seqs, offs, args.cpu_sample, WORKLOAD["scheme"], WORKLOAD["mode"])
        m = len(ref_score)
        if not (np.array_equal(ref_score, out["score"][:m]) and np.array_equal(ref_end, out["end"][:m])):
            raise SystemExit("GPU results differ from the CPU baseline on the sample")
        cpu.pop("seconds")
        cpu["parity_checked_triplets"] = m

    line = {
        "metric": METRIC, "value": value, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "int16x2" if st["lanes"] == 2 else "int32",
        "data": "synthetic: reference generator (bit-identical), 2-bit packed in HBM",
        "config": {"workload": f"{WORKLOAD['name']} {spec} rates {WORKLOAD['rates'][0]}:{WORKLOAD['rates'][1]} "
                               f"seed {WORKLOAD['seed']}, global, scheme 1/-1/-2 (linear gap)",
                   "triplets": n_total * world, "triplets_per_gpu": n_total, "cells": int(cells_all),
                   "parallelism": f"dp{world} (contiguous shards, weak scaling)",
                   "l2": "flushed (256 MiB write) between timed steps"},
        "triplets_per_s": trip_s,
        "failed_triplets": bad,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(st["launches"]) * args.steps,
        "clocks": clocks,
        "affine": aff,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
