#!/bin/bash
# shared-table hash draws in pac_mask (k_mask) and the sort-first pass 0 (build/variants/bt2): parity, A/B
mkdir -p gpurun_out
PAC_LIB=build/variants/bt2/libpac.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sort.py -m gpu -q --tb=short -x > gpurun_out/pytest_bt2.log 2>&1; tail -2 gpurun_out/pytest_bt2.log
for rep in 1 2; do
  python tools/bench_mask.py 100000000 | tail -1
  PAC_LIB=build/variants/bt2/libpac.so python tools/bench_mask.py 100000000 | tail -1
done
for rep in 1 2; do VARIANTS="default bt2" CONFIGS="C3" STEPS=50 bash tools/ab.sh; done
exit 0
