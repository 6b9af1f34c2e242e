#!/bin/bash
# default (dynamic copy-out, 32-row claims) against 64-row claims, pre-hash of odd warps, and both
mkdir -p gpurun_out
for rep in 1 2; do VARIANTS="default pre prec64" CONFIGS="C5" STEPS=20 bash tools/ab.sh; done
VARIANTS="default pre" CONFIGS="C2" STEPS=50 bash tools/ab.sh
exit 0
