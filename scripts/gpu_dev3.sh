#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -k design > gpurun_out/pytest_design.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_vs.log 2>&1
ST_NO_VSMALL=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_novs.log 2>&1
KB_TAG=_c bash scripts/kbench.sh
ST_CHUNK_MB=40 KB_TAG=_c40 bash scripts/kbench.sh
timeout 300 python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/prof3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc3d -s 3 -c 1 --csv \
  python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/prof3_dram.log 2>&1
