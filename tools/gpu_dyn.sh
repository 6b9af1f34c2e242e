#!/bin/bash
# dynamic copy-out claims (build/variants/dyn): parity, A/B on C5 / C2, phase clocks
mkdir -p gpurun_out
PAC_LIB=build/variants/dyn/libpac.so timeout 900 python -m pytest tests/test_gpu_lean.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -q --tb=short -x > gpurun_out/pytest_dyn.log 2>&1; tail -3 gpurun_out/pytest_dyn.log
for rep in 1 2; do VARIANTS="default dyn" CONFIGS="C5" STEPS=20 bash tools/ab.sh; done
VARIANTS="default dyn" CONFIGS="C2" STEPS=50 bash tools/ab.sh
PAC_LIB=build/variants/dynclk/libpac.so timeout 600 python tools/prof_agg.py --config C5 --rows 100000000 --iters 1 > gpurun_out/clk_dyn_C5.log 2>&1
grep LEANCLK gpurun_out/clk_dyn_C5.log | sort | tail -16
exit 0
