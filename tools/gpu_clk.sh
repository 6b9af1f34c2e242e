#!/bin/bash
# per-phase clock totals of k_agg_lean (CTA 0's warps; build/variants/clk = -DPAC_LEAN_CLK=1), C5 and C2 rows
mkdir -p gpurun_out
for c in "C5 --rows 100000000" "C2"; do
  set -- $c
  PAC_LIB=build/variants/clk/libpac.so timeout 600 python tools/prof_agg.py --config $c --iters 1 > gpurun_out/clk_$1.log 2>&1
  grep LEANCLK gpurun_out/clk_$1.log | sort | tail -16
done
exit 0
