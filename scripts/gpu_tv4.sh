#!/bin/bash
# tv2d sliced-chunk schedule: TV parity subset, K sweep, DRAM bytes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-tv4}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu -k "variants or coarse or solve_adjoint or design or fullsize or operator_parity" > gpurun_out/par_${TAG}.log 2>&1; tail -2 gpurun_out/par_${TAG}.log
{
for k in 0 4 8 12 16 24; do
  echo -n "K=$k 512^2x512 tv level 0 JAC: "; ST_CHUNK_K=$k python scripts/prof_op.py 2 0 2 512 512 tv 2>&1 | tail -1; done
echo -n "default 512^2x512 tv level 1 JAC: "; python scripts/prof_op.py 2 1 2 512 512 tv 2>&1 | tail -1
for lv in 0 1; do echo -n "default 256^3 tv level $lv JAC: "; python scripts/prof_op.py 2 $lv 2 256 256 tv 2>&1 | tail -1; done
for k in 0 8 16; do
  echo -n "DRAM K=$k 512^2 level 0: "
  ST_CHUNK_K=$k timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tv2d -s 3 -c 1 --csv python scripts/prof_op.py 2 0 2 512 512 tv 2>/dev/null | grep -o '"\(dram__bytes_[a-z]*.sum\|gpu__time_duration.sum\)","[^"]*","[^"]*"' | tr '\n' ' '; echo
done
} > gpurun_out/kb_${TAG}.log 2>&1
cat gpurun_out/kb_${TAG}.log
