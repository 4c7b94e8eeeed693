#!/bin/bash
# tc3r R = 4 / 5 (coefficient table), fine-level nu_pre = 0 (coarse correction of b + post-sweeps),
# 16-byte Krylov kernels: kernel times and benches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B=paper_2508_09589_b200
variant() { rm -f $B/build/tc3r.o; ST_NVCC_EXTRA="$1" python -c "from paper_2508_09589_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build failed: $1"; }
for R in 5 4; do
  variant "-DST_TC3R_R=$R"
  for m in 2 1 0; do echo -n "R=$R mode $m: "; timeout 300 python scripts/prof_op.py $m 0 3 64 128 tc c4 2>&1 | tail -1; done
done
bq() {  # $1 = tag, rest = bench args
  local tag=$1; shift
  timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bx_$tag.json 2> gpurun_out/bx_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/bx_$tag.json')); s=d['solver']; print('$tag', '$*', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'])" || tail -3 gpurun_out/bx_$tag.err
}
bq c4 --config 4
bq c4_02 --config 4 --nu-pre 0 --nu-post 2
bq c4_03 --config 4 --nu-pre 0 --nu-post 3
bq c2 --config 2
bq c2_02 --config 2 --nu-pre 0 --nu-post 2
bq c2_03 --config 2 --nu-pre 0 --nu-post 3
bq c33 --config 33
bq c33_02 --config 33 --nu-pre 0 --nu-post 2
bq c33_03 --config 33 --nu-pre 0 --nu-post 3
bq c3 --config 3
bq c3_02 --config 3 --nu-pre 0 --nu-post 2
bq c3_03 --config 3 --nu-pre 0 --nu-post 3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "prolongation or 3d" -p no:cacheprovider > gpurun_out/pytest_x.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_x.log
