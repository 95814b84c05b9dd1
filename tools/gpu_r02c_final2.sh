#!/bin/bash
# Round-2c evidence in one gpurun call (outputs under gpurun_out/final_c/).
F=gpurun_out/final_c2; mkdir -p $F
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > $F/pytest_gpu.log 2>&1; tail -2 $F/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $F/bench_c2.json 2> $F/bench_c2.err; tail -1 $F/bench_c2.json | cut -c1-300
timeout 900 python bench.py --impl reference > $F/bench_ref.json 2> $F/bench_ref.err; tail -1 $F/bench_ref.json | cut -c1-200
timeout 900 python tools/bench_modes.py > $F/configs.jsonl 2> $F/configs.err
timeout 900 python tools/bench_modes.py --affine >> $F/configs.jsonl 2>> $F/configs.err
(timeout 600 python tools/rows_c5.py; timeout 600 python tools/rows_c5.py -3) > $F/rows_c5.jsonl 2> $F/rows_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches.csv python bench.py --steps 2 --warmup 1 > $F/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wavefront_kernel --launch-skip 1 -c 1 -o $F/c5_1000_wave python tools/c5_one.py > $F/ncu_c5.log 2>&1; tail -1 $F/ncu_c5.log
wc -l $F/configs.jsonl $F/rows_c5.jsonl
