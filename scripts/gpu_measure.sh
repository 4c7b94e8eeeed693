#!/bin/bash
# parity subset + measurements: config 2/3/4 benches, config-2 launch list with DRAM bytes, ncu full of tc2d
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench3.log 2>&1; echo "rc=$?" >> gpurun_out/bench3.log
timeout 600 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 300 python scripts/prof_op.py 2 0 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2d -s 3 -c 2 -o gpurun_out/prof_tc2d \
  python scripts/prof_op.py 2 0 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu.log
