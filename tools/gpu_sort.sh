#!/bin/bash
# sort-first path: parity tests, C3 bench line, launch list of the C3 step
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sort.py -q -x --tb=short > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sort.log
tail -15 gpurun_out/pytest_sort.log
timeout 600 python bench.py --config C3 --steps 20 --no-cpu-baseline > gpurun_out/bench_sort_C3.json 2> gpurun_out/bench_sort_C3.err; echo "C3 rc=$?"; python tools/show_bench.py gpurun_out/bench_sort_C3.json; tail -3 gpurun_out/bench_sort_C3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_sort_C3.csv python tools/prof_agg.py --config C3 --iters 1 > gpurun_out/ncu_sort_launch.log 2>&1; echo "ncu rc=$?"
[ -n "$MORE" ] && timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_spill.py tests/test_gpu_fullsize.py -q -x --tb=short > gpurun_out/pytest_more.log 2>&1; tail -3 gpurun_out/pytest_more.log
exit 0
