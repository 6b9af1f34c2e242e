#!/bin/bash
# round-2 refresh: GPU parity suite, smoke, bench lines of every config, C3 sort-path launch list + ncu capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --tb=short --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"; python tools/show_bench.py gpurun_out/bench_default.json
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/show_bench.py gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C3.csv python bench.py --config C3 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_srt_" -c 20 -o gpurun_out/srt_C3_full -f python tools/prof_agg.py --config C3 --iters 1 > gpurun_out/ncu_srt_full.log 2>&1; echo "ncu full rc=$?"
exit 0
