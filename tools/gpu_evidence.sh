#!/bin/bash
# evidence pass: ncu --set full of k_agg_lean on C5 (1e8 rows) and C2 (full), the default bench's
# launch list, compute-sanitizer memcheck/racecheck logs
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_lean" -s 1 -c 1 -o gpurun_out/lean_C5 -f \
  python tools/prof_agg.py --config C5 --rows 100000000 --iters 2 > gpurun_out/ncu_lean_C5.log 2>&1; echo "ncu C5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_lean" -s 1 -c 1 -o gpurun_out/lean_C2 -f \
  python tools/prof_agg.py --config C2 --iters 2 > gpurun_out/ncu_lean_C2.log 2>&1; echo "ncu C2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_C5.log 2>&1; echo "ncu launches rc=$?"
[ -n "$SAN" ] && bash tools/sanitize.sh
exit 0
