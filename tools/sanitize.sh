#!/bin/bash
# compute-sanitizer memcheck and racecheck of the aggregation + finalize path on small inputs of
# each kernel family (C2: k_agg_tiles small-table instance; C5: k_agg_tiles_tm; C3: the HBM tier +
# k_spill_*; C4: k_agg_minmax), plus the opt-in k_agg_ws.  Logs in gpurun_out/sanitize_*.txt.
set -u
out=gpurun_out
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck; do
  for cfg in C2 C5 C3 C4; do
    rows=200000; [ $tool = racecheck ] && rows=40000
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/prof_agg.py --config $cfg --rows $rows --iters 1 \
      > $out/sanitize_${tool}_${cfg}.txt 2>&1
    echo "$tool $cfg rc=$?" | tee -a $out/sanitize_summary.txt
  done
  PAC_WS=1 timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/prof_agg.py --config C5 --rows 40000 --iters 1 \
    > $out/sanitize_${tool}_C5_ws.txt 2>&1
  echo "$tool C5 (PAC_WS=1) rc=$?" | tee -a $out/sanitize_summary.txt
  PAC_PART=1 timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/prof_agg.py --config C3 --rows 40000 --iters 1 \
    > $out/sanitize_${tool}_C3_part.txt 2>&1
  echo "$tool C3 (PAC_PART=1) rc=$?" | tee -a $out/sanitize_summary.txt
done
