#!/bin/bash
# A/B of the shared-table hash draws (build/variants/btab) against the default library
mkdir -p gpurun_out
PAC_LIB=build/variants/btab/libpac.so timeout 900 python -m pytest tests/test_gpu_lean.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -q --tb=short -x > gpurun_out/pytest_btab.log 2>&1; tail -3 gpurun_out/pytest_btab.log
for rep in 1 2; do
  VARIANTS="default btab" CONFIGS="C5" STEPS=20 bash tools/ab.sh
done
VARIANTS="default btab default btab" CONFIGS="C2" STEPS=50 bash tools/ab.sh
VARIANTS="default btab" CONFIGS="C1" STEPS=50 bash tools/ab.sh
exit 0
