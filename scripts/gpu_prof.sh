#!/bin/bash
# ncu --set full capture of the fine-level Jacobi sweep (config 2) + fp64 FMA peak probe.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
MODE=${MODE:-2}; LEVEL=${LEVEL:-0}
timeout 300 python scripts/prof_op.py $MODE $LEVEL > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tma2d -s 3 -c 2 -o gpurun_out/prof_jac \
  python scripts/prof_op.py $MODE $LEVEL > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu.log
