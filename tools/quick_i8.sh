#!/bin/bash
# Quick INT8 iteration on one GPU: the INT8 parity tests, then the C2 bench (INT8 only) per kernel variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "int8 or apply or c1 or stage or table3 or damped or e1" > gpurun_out/pytest_i8.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/pytest_i8.log
for V in ${VARIANTS:-tmem}; do
  OVX_I8_KERNEL=$V timeout 300 python bench.py --no-cpu-baseline --no-fp64-companion > gpurun_out/bench_$V.json 2>gpurun_out/bench_$V.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$V.json'));print('$V', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],4))" || tail -5 gpurun_out/bench_$V.err
done
