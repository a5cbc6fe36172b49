#!/bin/bash
# One GPU round: parity tests, smoke, microbench, bench (both paths), launch list.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 120 ./tools/microbench > gpurun_out/microbench.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_int8.json 2> gpurun_out/bench_int8.err
timeout 600 python bench.py --path fp64 --no-cpu-baseline > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/bench_int8.json gpurun_out/bench_fp64.json
