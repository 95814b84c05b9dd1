#!/bin/bash
# End-of-round GPU evidence in one gpurun call: GPU tests, smoke, bench line,
# secondary configs and full-size configs (outputs under gpurun_out/).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-300
timeout 900 python tools/bench_modes.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 900 python tools/bench_modes.py --affine >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
timeout 900 python tools/full_configs.py > gpurun_out/full_configs.jsonl 2> gpurun_out/full_configs.err
wc -l gpurun_out/configs.jsonl gpurun_out/full_configs.jsonl
