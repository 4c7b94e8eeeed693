#!/bin/bash
# ncu --set full of the config-3-shaped (256^3, space-time design) level-0 and level-1 Jacobi sweeps (tv2d)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-tv}
for lv in 0 1; do
  timeout 300 python scripts/prof_op.py 2 $lv 2 256 256 tv > gpurun_out/prof_${TAG}_l${lv}_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tv2d -s 3 -c 1 -o gpurun_out/prof_${TAG}_l${lv} \
    python scripts/prof_op.py 2 $lv 2 256 256 tv > gpurun_out/prof_${TAG}_l${lv}_ncu.log 2>&1
  echo "rc=$?" >> gpurun_out/prof_${TAG}_l${lv}_ncu.log
done
