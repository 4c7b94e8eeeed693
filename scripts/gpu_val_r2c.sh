#!/bin/bash
# dense coarsest on the free nodes, PDL launches, tc3r at 128 registers (2 CTAs/SM), tv2d fine-level PRO:
# kernel times, benches, GPU suite
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
for m in 2 1 0; do echo -n "tc3r mode $m: "; timeout 300 python scripts/prof_op.py $m 0 3 64 128 tc c4 2>&1 | tail -1; done
bq() {  # $1 = tag, rest = bench args
  local tag=$1; shift
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bx_$tag.json 2> gpurun_out/bx_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/bx_$tag.json')); s=d['solver']; print('$tag', '$*', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'], 'launches', d.get('gpu_launches'))" || tail -3 gpurun_out/bx_$tag.err
}
bq c4 --config 4
bq c2 --config 2
bq c33 --config 33
bq c5 --config 5
bq c3 --config 3
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
