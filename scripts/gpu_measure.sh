#!/bin/bash
# measurement call: config-2 bench + launch list + ncu full of the fine sweep; configs 3/4 timing
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench3.log 2>&1; echo "rc=$?" >> gpurun_out/bench3.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 300 python scripts/prof_op.py 2 0 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2d -s 3 -c 2 -o gpurun_out/prof_tc2d \
  python scripts/prof_op.py 2 0 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu.log
