#!/bin/bash
# C4: MIN/MAX parity tests on the default build, then k_agg_minmax_p vs _v (PAC_NO_MMP) vs variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "minmax or MIN or MAX or nonfinite or C4 or fullsize or determinism or small_tables" > gpurun_out/pytest_c4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_c4.log
one() {  # name, env...
  local n=$1; shift
  env "$@" timeout 600 python bench.py --config C4 --steps 50 --no-cpu-baseline > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$n.json').read().strip().splitlines()[-1]); r=d['roofline']
print('%-10s %.3g rows/s  kernel %.3f ms  frac %.3f  step %.3f ms  %s'%('$n',d['value'],r['kernel_ms'],r['frac'],d['ms_per_step'],r['kernel']))" || tail -3 gpurun_out/ab_$n.err
}
for r in 1 2; do
  one p PAC_X=1
  one v PAC_NO_MMP=1
  for v in ${VARS}; do one $v PAC_LIB=build/variants/$v/libpac.so; done
done
