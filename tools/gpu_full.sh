#!/bin/bash
# full parity suite + C5/C2 bench lines (+ optional ncu capture of k_agg_lean on C5)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in C5 C2; do timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python tools/show_bench.py gpurun_out/bench_$c.json; done
if [ -n "$NCU" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_lean" -s 1 -c 1 -o gpurun_out/lean_C5 -f python tools/prof_agg.py --config C5 --rows 100000000 --iters 2 > gpurun_out/ncu_lean.log 2>&1; echo "ncu rc=$?"; fi
