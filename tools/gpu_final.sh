#!/bin/bash
# end-of-round evidence: parity suite, smoke, every bench line (+ the reference arm), the C5 launch
# list, ncu --set full of the C4 kernel (cp.async-staged k_agg_minmax_v)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"; python tools/show_bench.py gpurun_out/bench_C5.json
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python tools/show_bench.py gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_minmax_v" -s 1 -c 1 -o gpurun_out/mmv_C4 -f \
  python tools/prof_agg.py --config C4 --iters 2 > gpurun_out/ncu_mmv_C4.log 2>&1; echo "ncu C4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_C5.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C4.csv \
  python bench.py --config C4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_C4.log 2>&1; echo "ncu C4 launches rc=$?"
exit 0
