#!/bin/bash
# parity suite + C2 timing + one ncu capture of k_agg_tiles (instruction counts)
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E |___ test|passed|failed" | head -20
python tools/prof_agg.py --config C2 --iters 4 --gcap 16 > gpurun_out/prof_plain.log 2>&1 && tail -2 gpurun_out/prof_plain.log && \
ncu --set full --clock-control none --import-source on -k regex:"k_agg_tiles" -s 1 -c 1 -o gpurun_out/prof_cur -f python tools/prof_agg.py --config C2 --iters 2 --gcap 16 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
