#!/bin/bash
# CLI end to end on C2: generate FASTA, then `trioalign align` with phase timings
# (TA_PROFILE_CLI: parse / plan / run_batch / format; TA_PROFILE_PIPELINE: the
# engine's pipelined one-shot call).
set -e
B=paper_2605_28400_b200/trioalign
mkdir -p /tmp/cli_c2
[ -f /tmp/cli_c2/c2.fa ] || $B generate --spec fixed:150:150:150:1000000 --rates 0.025:0.005 --seed 2 --out /tmp/cli_c2/c2.fa
ls -la /tmp/cli_c2/c2.fa
for i in 1 2; do
  s=$(date +%s%N)
  TA_PROFILE_CLI=1 TA_PROFILE_PIPELINE=1 $B align --in /tmp/cli_c2/c2.fa --out /tmp/cli_c2/out.csv --mode global 2>&1 | grep -v "] chunk" || true
  e=$(date +%s%N)
  echo "align wall $(( (e - s) / 1000000 )) ms"
done
head -3 /tmp/cli_c2/out.csv
