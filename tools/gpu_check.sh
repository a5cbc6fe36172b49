#!/bin/bash
# One GPU round: parity tests, smoke, microbench, bench (all paths), launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 120 ./tools/microbench > gpurun_out/microbench.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for p in int8 fp64 fp64_dense; do
  timeout 600 python bench.py --path $p $( [ $p != int8 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err
done
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/microbench.jsonl
for p in int8 fp64 fp64_dense; do python -c "import json;d=json.load(open('gpurun_out/bench_$p.json'));print('$p', '%.3e'%d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
