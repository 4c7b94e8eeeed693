#!/bin/bash
# tv2d (padded k~ table): TV parity subset, level timings (L2 promotion x chunk), DRAM bytes, ncu of level 0
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-tv3}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu -k "variants or coarse or solve_adjoint or design or fullsize or operator_parity" > gpurun_out/par_${TAG}.log 2>&1; tail -2 gpurun_out/par_${TAG}.log
{
for pr in 128 0 64; do for k in 0 16; do for lv in 0 1; do
  echo -n "promo=$pr K=$k 512^2x512 tv level $lv JAC: "; ST_L2PROMO=$pr ST_CHUNK_K=$k python scripts/prof_op.py 2 $lv 2 512 512 tv 2>&1 | tail -1; done; done; done
for pr in 128 0; do for lv in 0 1; do echo -n "promo=$pr 256^3 tv level $lv JAC: "; ST_L2PROMO=$pr python scripts/prof_op.py 2 $lv 2 256 256 tv 2>&1 | tail -1; done; done
for cfg in "128 0" "0 0" "0 16"; do set -- $cfg
  echo -n "DRAM promo=$1 K=$2 512^2 level 0: "
  ST_L2PROMO=$1 ST_CHUNK_K=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tv2d -s 3 -c 1 --csv python scripts/prof_op.py 2 0 2 512 512 tv 2>/dev/null | grep -o '"\(dram__bytes_[a-z]*.sum\|gpu__time_duration.sum\)","[^"]*","[^"]*"' | tr '\n' ' '; echo
done
} > gpurun_out/kb_${TAG}.log 2>&1
cat gpurun_out/kb_${TAG}.log
TAG=$TAG bash scripts/gpu_prof_tv.sh
