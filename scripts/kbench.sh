#!/bin/bash
# kernel microbenchmarks: config-2 levels 0/1 all modes; config-3-shaped fine level; config-4 fine level
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{
for lv in 0 1; do for m in 0 1 2 3; do echo -n "cfg2 level $lv mode $m: "; python scripts/prof_op.py $m $lv 2>&1 | tail -1; done; done
for lv in 0 1; do echo -n "cfg3-shaped 256^3 tv level $lv JAC: "; python scripts/prof_op.py 2 $lv 2 256 256 tv 2>&1 | tail -1; done
for lv in 0 1 2; do echo -n "cfg4 64^3x128 level $lv JAC: "; python scripts/prof_op.py 2 $lv 3 64 128 tc c4 2>&1 | tail -1; done
} > gpurun_out/kbench${KB_TAG}.log 2>&1
