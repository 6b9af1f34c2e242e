#!/bin/bash
# round-robin quarter balancing of the owner mode (build/variants/q2): parity, A/B on C5, phase clocks
mkdir -p gpurun_out
PAC_LIB=build/variants/q2/libpac.so timeout 900 python -m pytest tests/test_gpu_lean.py tests/test_gpu_determinism.py -m gpu -q --tb=short -x > gpurun_out/pytest_q2.log 2>&1; tail -3 gpurun_out/pytest_q2.log
for rep in 1 2; do VARIANTS="default q2" CONFIGS="C5" STEPS=20 bash tools/ab.sh; done
PAC_LIB=build/variants/q2clk/libpac.so timeout 600 python tools/prof_agg.py --config C5 --rows 100000000 --iters 1 > gpurun_out/clk_q2_C5.log 2>&1
grep LEANCLK gpurun_out/clk_q2_C5.log | sort | tail -16
exit 0
