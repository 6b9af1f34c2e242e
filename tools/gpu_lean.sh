#!/bin/bash
# lean-kernel iteration: parity tests, C5/C2 bench lines, one ncu capture of k_agg_lean on C5
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lean.py -q -x --tb=short > gpurun_out/pytest_lean.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lean.log
tail -5 gpurun_out/pytest_lean.log
if [ -n "$MORE" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small_tables.py tests/test_gpu_nonfinite.py tests/test_gpu_determinism.py tests/test_gpu_tm.py -q -x --tb=short > gpurun_out/pytest_more.log 2>&1; echo "pytest more rc=$?" >> gpurun_out/pytest_more.log; tail -3 gpurun_out/pytest_more.log; fi
for c in C5 C2 C1; do timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_lean_$c.json 2> gpurun_out/bench_lean_$c.err; echo "$c rc=$?"; python tools/show_bench.py gpurun_out/bench_lean_$c.json 2>/dev/null || tail -c 600 gpurun_out/bench_lean_$c.json; done
if [ -n "$NCU" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_lean" -s 1 -c 1 -o gpurun_out/lean_C5 -f python tools/prof_agg.py --config C5 --rows 100000000 --iters 2 > gpurun_out/ncu_lean.log 2>&1; echo "ncu rc=$?"; fi
