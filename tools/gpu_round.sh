#!/bin/bash
# One full GPU validation pass: parity tests, smoke, the default bench line (INT8, with the CPU
# baseline), the FP64 bench, the launch list of the bench command, the step_i8ws phase trace and the
# TMEM throughput microbenchmark.  Results under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_int8.json 2> gpurun_out/bench_int8.err
timeout 300 python bench.py --path fp64 --no-cpu-baseline > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
[ -f tools/abl/libovx_trace.so ] && timeout 120 python tools/trace_ws.py > gpurun_out/trace_ws.txt 2>&1
[ -x tools/tmem_bench ] && timeout 60 ./tools/tmem_bench > gpurun_out/tmem_bench.jsonl 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
python -c "import json;d=json.load(open('gpurun_out/bench_int8.json'));print('int8', d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
tail -6 gpurun_out/trace_ws.txt
