#!/bin/bash
# tc3d stored-stencil variants at 1 / 2 CTAs per SM (config-4 levels 1-3, config-4 bench); ncu --set full of
# the config-4 fine sweep (tc3r, two CTAs per SM)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B=paper_2508_09589_b200
variant() { rm -f $B/build/tc3d.o; ST_NVCC_EXTRA="$1" python -c "from paper_2508_09589_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build failed: $1"; }
for v in "-DST_TC3D_MINB1=2" "-DST_TC3D_MINB1=1"; do
  variant "$v"
  for lv in 1 2 3; do echo -n "$v level $lv JAC: "; timeout 300 python scripts/prof_op.py 2 $lv 3 64 128 tc c4 2>&1 | tail -1; done
  timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bm.json 2> gpurun_out/bm.err
  python -c "import json; d=json.load(open('gpurun_out/bm.json')); s=d['solver']; print('$v config 4', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'])" || tail -3 gpurun_out/bm.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3r -s 3 -c 1 -o gpurun_out/ncu_tc3r_2cta \
  python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/ncu_tc3r_2cta.log 2>&1; echo "ncu tc3r rc=$?"
rm -f paper_2508_09589_b200/build/tc3d.o; python -c "from paper_2508_09589_b200 import build as b; b.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_schedules.py -m gpu -q -x -k "pde_filter" -p no:cacheprovider > gpurun_out/pytest_pf.log 2>&1; echo "pytest pde filter rc=$?"; tail -1 gpurun_out/pytest_pf.log
for k in 1 2; do timeout 600 python bench.py --config 2 > gpurun_out/c2_rerun_$k.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/c2_rerun_$k.json')); s=d['solver']; print('config 2 rerun', round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), s['fwd_ms'], s['setup_ms'])"; done
