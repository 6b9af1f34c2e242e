#!/bin/bash
# parity suite + C2 bench line + one ncu --set full capture of k_agg_tiles (C2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_C2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('C2 %.3g rows/s  kernel %.3f ms  frac %.3f  step %.3f ms'%(d['value'],r['kernel_ms'],r['frac'],d['ms_per_step']))"
for c in ${EXTRA_CONFIGS}; do timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c %.3g rows/s  kernel %.3f ms  frac %.3f  step %.3f ms'%(d['value'],r['kernel_ms'],r['frac'],d['ms_per_step']))"; done
if [ -n "$NCU" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_agg_tiles" -s 1 -c 1 -o gpurun_out/agg_C2 -f python tools/prof_agg.py --config C2 --iters 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; fi
