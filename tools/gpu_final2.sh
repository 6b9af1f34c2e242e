#!/bin/bash
# end-of-round evidence (after the dynamic copy-out): parity suite, smoke, every bench line (+ the
# reference arm), ncu --set full of k_agg_lean on C5 (1e8 rows) and C2, the default bench's launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"; python tools/show_bench.py gpurun_out/bench_C5.json
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python tools/show_bench.py gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_lean" -s 1 -c 1 -o gpurun_out/lean_C5 -f \
  python tools/prof_agg.py --config C5 --rows 100000000 --iters 2 > gpurun_out/ncu_lean_C5.log 2>&1; echo "ncu C5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_lean" -s 1 -c 1 -o gpurun_out/lean_C2 -f \
  python tools/prof_agg.py --config C2 --iters 2 > gpurun_out/ncu_lean_C2.log 2>&1; echo "ncu C2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_C5.log 2>&1; echo "ncu launches rc=$?"
exit 0
