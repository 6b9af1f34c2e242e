#!/bin/bash
# ncu --set full captures of the sort-first kernels on C3 (1e8 rows)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_srt_(scatter|agg|hash)" -c 6 -o gpurun_out/srt_C3 -f \
  python tools/prof_agg.py --config C3 --iters 1 > gpurun_out/ncu_srt.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_srt.log
exit 0
