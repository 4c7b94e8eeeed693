#!/bin/bash
# A/B: fine-level prolongation fusion (tv2d PRO, since removed) on / off and PDL on / off on configs 3, 33, 2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B=paper_2508_09589_b200
full() { rm -rf $B/build; ST_NVCC_EXTRA="$1" python -c "from paper_2508_09589_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build failed: $1"; }
bq() {  # $1 = tag, rest = bench args
  local tag=$1; shift
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$tag.json')); s=d['solver']; print('$tag', '$*', round(d['value']/1e6,1), 'MDOF/s fwd_ms', s['fwd_ms'], 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$tag.err
}
full ""
bq c33_pro1 --config 33 --fuse-prolong 1
bq c33_pro0 --config 33 --fuse-prolong 0
bq c3_pro1 --config 3 --fuse-prolong 1
bq c3_pro0 --config 3 --fuse-prolong 0
bq c2_pdl --config 2
full "-DST_NO_PDL"
bq c2_nopdl --config 2
bq c33_nopdl --config 33 --fuse-prolong 1
bq c3_nopdl --config 3 --fuse-prolong 1
