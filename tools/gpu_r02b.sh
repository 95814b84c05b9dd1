mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-600
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wavefront_kernel -c 1 -o gpurun_out/glob_src -f python tools/prof_one.py fixed:150:150:150:40000 0.025 0.005 2 0 1 > gpurun_out/ncu_glob.log 2>&1; tail -2 gpurun_out/ncu_glob.log
