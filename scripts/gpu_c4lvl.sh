#!/bin/bash
# matrix-free time-coarsened (3+1)D level (tc3r on level 1) + paired time-transfer kernels:
# transfer / coarse-operator / 3D parity tests, slab tests, benches of configs 4 and 2, config-4 launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-i}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_schedules.py "tests/test_gpu_fullsize.py::test_fullsize_solution_certified_by_oracle_rows[config4]" "tests/test_gpu_fullsize.py::test_fullsize_solution_certified_by_oracle_rows[config2]" -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_3d_$TAG.log 2>&1; echo "pytest 3d rc=$?"; tail -3 gpurun_out/pytest_3d_$TAG.log
for c in 4 2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bi_c$c.json 2> gpurun_out/bi_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bi_c$c.json')); s=d['solver']; e=d['e2e']; print('config $c', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms e2e', round(e['value']/1e6,1), 'its', s['fwd_its'], s['adj_its'], 'setup', s['setup_ms'], 'clk', d['clocks']['sm_mhz'], d['clocks'].get('reasons'))" || tail -5 gpurun_out/bi_c$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/launches_c4_$TAG.csv \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c4_$TAG.log 2>&1; echo "ncu launch rc=$?"
