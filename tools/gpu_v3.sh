#!/bin/bash
# default (committed) against: claim address hoisted (hoist), + B outputs published by five warps (pub), + 64-row claims (pub64)
mkdir -p gpurun_out
PAC_LIB=build/variants/pub/libpac.so timeout 900 python -m pytest tests/test_gpu_lean.py tests/test_gpu_determinism.py -m gpu -q --tb=short -x > gpurun_out/pytest_pub.log 2>&1; tail -2 gpurun_out/pytest_pub.log
for rep in 1 2; do VARIANTS="default pub pub64" CONFIGS="C5" STEPS=20 bash tools/ab.sh; done
exit 0
