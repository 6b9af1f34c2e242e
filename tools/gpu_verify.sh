#!/bin/bash
# end-of-round verification: the GPU parity suite, smoke(), and the default bench line
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q --tb=short -x ) > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json; tail -4 gpurun_out/bench_default.err
exit 0
