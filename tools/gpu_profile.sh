#!/bin/bash
# ncu captures of the step kernel (one GPU): full set for the given path(s), plus a launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
for p in ${PATHS:-int8 fp64}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 3 -c 1 \
     -o gpurun_out/prof_${p}_${TAG} -f python bench.py --path $p --steps 2 --warmup 3 --no-cpu-baseline \
     > gpurun_out/prof_${p}_${TAG}.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -c 12 --csv --log-file gpurun_out/launches_${p}_${TAG}.csv python bench.py --path $p --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out
