#!/bin/bash
# C4 staging A/B: MIN/MAX parity tests, then default vs variants interleaved
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "minmax or MIN or MAX or nonfinite or C4 or fullsize or determinism" > gpurun_out/pytest_c4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_c4.log
for r in 1 2; do VARIANTS="default ${VARS:-nostage head}" CONFIGS="C4" STEPS=50 bash tools/ab.sh; done
