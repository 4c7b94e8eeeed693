#!/bin/bash
# development GPU call: parity tests, bench, smoother sweep
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$SWEEP" ]; then timeout 900 python scripts/sweep_smoother.py $SWEEP > gpurun_out/sweep.log 2>&1; fi
