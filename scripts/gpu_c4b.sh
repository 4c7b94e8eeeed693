#!/bin/bash
# 3D space prolongation kernel + paired time transfers + matrix-free time levels: parity / slab tests,
# config-4 parameter runs, ncu of the stored-stencil 3D level
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-j}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "transfer or coarse_operators" > gpurun_out/pytest_tr_$TAG.log 2>&1; echo "pytest transfer rc=$?"; tail -3 gpurun_out/pytest_tr_$TAG.log
run() { # label, args...
  local lab=$1; shift
  timeout 600 python bench.py --config 4 --no-cpu-baseline --e2e-steps 0 --steps 3 "$@" > gpurun_out/bj_$lab.json 2> gpurun_out/bj_$lab.err
  python -c "import json; d=json.load(open('gpurun_out/bj_$lab.json')); s=d['solver']; print('c4 $lab', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'])" || tail -3 gpurun_out/bj_$lab.err
}
run base
run nc6 --nu-coarse 6
run nc7 --nu-coarse 7
run r10 --restart 10
run r30 --restart 30
run gm --krylov gmres
run nf4m --nu-fine-nodes 4000000
for a in "2 0" "2 1" "2 2"; do timeout 300 python scripts/prof_op.py $a 3 64 128 tc c4; done
timeout 300 python scripts/prof_op.py 2 1 3 64 128 tc
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3d_kernel -s 3 -c 1 -o gpurun_out/ncu_tc3d_l1_$TAG \
  python scripts/prof_op.py 2 1 3 64 128 tc c4 > gpurun_out/ncu_tc3d_l1_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x --timeout 600 -p no:cacheprovider --deselect tests/test_gpu_parity.py::test_coarse_operators > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
