#!/bin/bash
# faster per-design Gershgorin bound (tv2d fine level) and marching sensitivities: GPU suite, smoke, benches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
for c in 3 5 2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bd_c$c.json 2> gpurun_out/bd_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bd_c$c.json')); s=d['solver']; print('config $c', round(d['value']/1e6,1), 'MDOF/s e2e', round(d['e2e']['value']/1e6,1), 'setup', s['setup_ms'], 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bd_c$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gersh|sens" -c 20 --csv --log-file gpurun_out/launches_setup_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo "ncu rc=$?"
