#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -k design > gpurun_out/pytest_design.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/pytest_parity.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench5.log 2>&1
timeout 300 python scripts/prof_op.py 2 0 2 256 256 tv > gpurun_out/prof_tv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tv2d -s 3 -c 1 -o gpurun_out/prof_tv2d \
  python scripts/prof_op.py 2 0 2 256 256 tv > gpurun_out/prof_tv_ncu.log 2>&1
