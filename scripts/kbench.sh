#!/bin/bash
# kernel microbenchmarks: config-2 level operators, all modes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lv in 0 1; do for m in 0 1 2 3; do echo -n "level $lv mode $m: "; python scripts/prof_op.py $m $lv 2>&1 | tail -1; done; done > gpurun_out/kbench.log 2>&1
