mkdir -p gpurun_out/ab2 gpurun_out/c5
timeout 900 python -m pytest tests/test_gpu_affine.py -x -q > gpurun_out/ab2/pytest_aff.log 2>&1; tail -2 gpurun_out/ab2/pytest_aff.log
bash tools/gpu_ab.sh "--n 200000 --c4 20000 --gap-open -3" base2 tree > gpurun_out/ab2/ab.jsonl 2>&1; cat gpurun_out/ab2/ab.jsonl | cut -c1-160
timeout 120 python tools/c5_one.py > gpurun_out/c5/plain.txt 2>&1; cat gpurun_out/c5/plain.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wavefront_kernel --launch-skip 1 -c 1 -o gpurun_out/c5/c5_1000 python tools/c5_one.py > gpurun_out/c5/ncu.log 2>&1; tail -3 gpurun_out/c5/ncu.log
