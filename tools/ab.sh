#!/bin/bash
# A/B of libpac variants on bench configs: VARIANTS="default minb2" CONFIGS="C2 C5" bash tools/ab.sh
for v in ${VARIANTS:-default}; do
  for c in ${CONFIGS:-C2}; do
    if [ "$v" = default ]; then L=""; else L="build/variants/$v/libpac.so"; fi
    PAC_LIB=$L timeout 600 python bench.py --config $c --steps ${STEPS:-20} --no-cpu-baseline > gpurun_out/ab_${v}_$c.json 2> gpurun_out/ab_${v}_$c.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_${v}_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('%-10s $c %.3g rows/s  kernel %.3f ms  frac %.3f  step %.3f ms'%('$v',d['value'],r['kernel_ms'],r['frac'],d['ms_per_step']))" || tail -3 gpurun_out/ab_${v}_$c.err
  done
done
