mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-400
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wavefront_kernel -c 1 -o gpurun_out/prof_t8 python tools/prof_one.py fixed:250:250:250:20000 0.025 0.005 3 0 1 > gpurun_out/prof_t8.log 2>&1; tail -2 gpurun_out/prof_t8.log
