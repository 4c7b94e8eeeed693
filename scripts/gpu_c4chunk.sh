#!/bin/bash
# (3+1)D config-4 fine sweep (tc3d) vs plane-chunk size (balanced chunks), with DRAM bytes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for k in 0 8 16 32 64; do
  echo -n "K=$k config4 level 0 JAC: "; ST_CHUNK_K=$k python scripts/prof_op.py 2 0 3 64 128 tc c4 2>&1 | tail -1
done
for k in 0 16; do
  echo -n "DRAM K=$k: "
  ST_CHUNK_K=$k timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc3d -s 3 -c 1 --csv python scripts/prof_op.py 2 0 3 64 128 tc c4 2>/dev/null | grep -o '"\(dram__bytes_[a-z]*.sum\|gpu__time_duration.sum\)","[^"]*","[^"]*"' | tr '\n' ' '; echo
done
