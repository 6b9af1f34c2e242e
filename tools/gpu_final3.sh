#!/bin/bash
# last pass of the round: full parity suite, smoke, pac_mask alone, the default bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python tools/bench_mask.py 100000000 | tee gpurun_out/bench_mask.txt | tail -1
python tools/bench_mask.py 60000000 | tee -a gpurun_out/bench_mask.txt | tail -1
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"; python tools/show_bench.py gpurun_out/bench_C5.json
exit 0
