#!/bin/bash
# Round-2c last check on the final tree: GPU tests, smoke, bench line, configs.
F=gpurun_out/last_c2; mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -x -q > $F/pytest_gpu.log 2>&1; tail -2 $F/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $F/bench_c2.json 2> $F/bench_c2.err; tail -1 $F/bench_c2.json | cut -c1-200
timeout 900 python tools/bench_modes.py > $F/configs.jsonl 2> $F/configs.err
timeout 900 python tools/bench_modes.py --affine >> $F/configs.jsonl 2>> $F/configs.err
wc -l $F/configs.jsonl
