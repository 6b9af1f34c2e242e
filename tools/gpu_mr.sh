#!/bin/bash
# mode P ranks by match_any for <= 8 slots (build/variants/mr): parity, A/B on C2 (and C5 as the control)
mkdir -p gpurun_out
PAC_LIB=build/variants/mr/libpac.so timeout 900 python -m pytest tests/test_gpu_lean.py tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_small_tables.py -m gpu -q --tb=short -x > gpurun_out/pytest_mr.log 2>&1; tail -2 gpurun_out/pytest_mr.log
for rep in 1 2; do VARIANTS="default mr" CONFIGS="C2" STEPS=50 bash tools/ab.sh; done
VARIANTS="default mr" CONFIGS="C5" STEPS=10 bash tools/ab.sh
exit 0
