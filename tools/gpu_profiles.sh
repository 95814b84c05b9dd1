#!/bin/bash
# ncu evidence for profiles/ in one gpurun call (outputs under gpurun_out/prof/):
# full C2 launch of the global kernel (summary + DRAM traffic), traceback
# wavefront + walker on a C2 chunk, affine global on a C2 prefix, and the
# launch list of a short bench run.
mkdir -p gpurun_out/prof
P=gpurun_out/prof
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:wavefront_kernel -s 1 -c 1 -o $P/glob_full -f python tools/prof_run.py --triplets 1000000 --runs 2 > $P/glob_full.log 2>&1; tail -1 $P/glob_full.log
timeout 600 $NCU -k regex:"wavefront_kernel|walker" -s 2 -c 2 -o $P/rows -f python tools/prof_run.py --rows --triplets 6000 --runs 2 > $P/rows.log 2>&1; tail -1 $P/rows.log
timeout 600 $NCU -k regex:affine_kernel -s 0 -c 1 -o $P/affine -f python tools/prof_aff1.py > $P/affine.log 2>&1; tail -1 $P/affine.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $P/bench_under_ncu.log 2>&1; tail -1 $P/launches.csv | cut -c1-200
