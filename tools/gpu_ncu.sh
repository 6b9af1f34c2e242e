#!/bin/bash
# one ncu --set full capture (outputs stay below gpurun's 64 MiB copy-back limit): CFG=C2|C5
mkdir -p gpurun_out
CFG=${CFG:-C2}
K=${KREGEX:-k_agg_tiles}
ROWS=${ROWS:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/agg_$CFG -f \
  python tools/prof_agg.py --config $CFG --rows $ROWS --iters 2 > gpurun_out/ncu_full_$CFG.log 2>&1; echo "ncu $CFG rc=$?"
ls -la gpurun_out/agg_$CFG.ncu-rep
