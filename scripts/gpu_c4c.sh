#!/bin/bash
# tc3d stored-stencil FMA chains (4 / 8) on the config-4 levels 1-2, restart-length runs of configs 4 and 2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-l}
run() { # config, label, args...
  local c=$1 lab=$2; shift 2
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 3 "$@" > gpurun_out/bl_$lab.json 2> gpurun_out/bl_$lab.err
  python -c "import json; d=json.load(open('gpurun_out/bl_$lab.json')); s=d['solver']; print('c$c $lab', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'])" || tail -3 gpurun_out/bl_$lab.err
}
for nch in 8 2 4; do
  touch paper_2508_09589_b200/csrc/tc3d.cu
  ST_NVCC_EXTRA="-DST_TC3D_NCH=$nch" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
  echo "== NCH $nch"
  for a in "2 1" "2 2" "1 1"; do timeout 300 python scripts/prof_op.py $a 3 64 128 tc c4; done
  run 4 nch$nch
done
# (the library is now the default build, NCH = 4)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "coarse_operators or test_operator_parity or solve_parity or config4 or cfg4" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
run 4 r8 --restart 8
run 4 r10 --restart 10
run 4 r12 --restart 12
run 2 c2base
run 2 c2r8 --restart 8
run 2 c2r10 --restart 10
run 2 c2r12 --restart 12
