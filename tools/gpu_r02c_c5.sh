#!/bin/bash
# Round-2c wave-mode A/B: C5 score (all modes) and rows, variant builds vs the tree; wave / parity GPU tests.
F=gpurun_out/c5ab; mkdir -p $F
for v in "$@"; do
  if [ "$v" = tree ]; then E=""; else E="TA_LIB_PATH_EXPERIMENT=exp/$v/libtrioalign_b200.so"; fi
  env $E TA_WAVE_DELAY=$v timeout 300 python tools/c5_probe.py >> $F/c5.jsonl 2>> $F/c5.err
  env $E timeout 300 python tools/rows_c5.py > $F/rows_$v.jsonl 2>> $F/c5.err
done
cat $F/c5.jsonl | cut -c1-200; head -5 $F/rows_*.jsonl | cut -c1-200
timeout 1200 python -m pytest tests/test_gpu_wave_coresidency.py tests/test_gpu_parity.py tests/test_gpu_config_parity.py -x -q > $F/pytest.log 2>&1; tail -2 $F/pytest.log
