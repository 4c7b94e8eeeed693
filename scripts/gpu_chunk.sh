#!/bin/bash
# tv2d plane-chunk x tile-order sweep (balanced chunks, cross-segment prefetch) + DRAM bytes per launch
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-ck}
{
for o in 0 1; do for k in 0 12 16 24 32; do
  echo -n "order=$o K=$k 512^2x512 tv level 0 JAC: "; ST_TILE_ORDER=$o ST_CHUNK_K=$k python scripts/prof_op.py 2 0 2 512 512 tv 2>&1 | tail -1; done
  echo -n "order=$o K=0 512^2x512 tv level 1 JAC: "; ST_TILE_ORDER=$o python scripts/prof_op.py 2 1 2 512 512 tv 2>&1 | tail -1
  for k in 0 16; do echo -n "order=$o K=$k 256^3 tv level 0 JAC: "; ST_TILE_ORDER=$o ST_CHUNK_K=$k python scripts/prof_op.py 2 0 2 256 256 tv 2>&1 | tail -1; done
done
for cfg in "0 0" "0 16" "1 16" "1 0"; do set -- $cfg
  echo -n "DRAM order=$1 K=$2 512^2 level 0: "
  ST_TILE_ORDER=$1 ST_CHUNK_K=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tv2d -s 3 -c 1 --csv python scripts/prof_op.py 2 0 2 512 512 tv 2>/dev/null | grep -o '"\(dram__bytes_[a-z]*.sum\|gpu__time_duration.sum\)","[^"]*","[^"]*"' | tr '\n' ' '; echo
done
} > gpurun_out/kb_${TAG}.log 2>&1
cat gpurun_out/kb_${TAG}.log
