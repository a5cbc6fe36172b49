cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash tools/gpu_check.sh
for ey in 4 8; do OVX_I8_EY=$ey timeout 300 python bench.py --no-cpu-baseline --no-fp64-companion > gpurun_out/bench_int8_ey$ey.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_int8_ey$ey.json'));print('EY=$ey', d['ms_per_step'], d['roofline']['frac'])"; done
PATHS="int8" TAG=v9 bash tools/gpu_profile.sh > /dev/null 2>&1
