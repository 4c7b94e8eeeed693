#!/bin/bash
# A/B: tc2d with 4 vs 5 resident CTAs; kernel microbenchmarks; ncu full of the (3+1)D kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
KB_TAG=_m4 bash scripts/kbench.sh
ST_LIB_PATH=$PWD/paper_2508_09589_b200/libst_m5.so KB_TAG=_m5 bash scripts/kbench.sh
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_m4.log 2>&1
ST_LIB_PATH=$PWD/paper_2508_09589_b200/libst_m5.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_m5.log 2>&1
timeout 300 python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/prof3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc3d -s 3 -c 1 -o gpurun_out/prof_tc3d \
  python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/prof3_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof3_ncu.log
