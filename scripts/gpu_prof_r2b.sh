#!/bin/bash
# evidence: config-4 launch list (tc3r), ncu --set full of the config-4 fine sweep (tc3r R = 5) and of the
# 512^2 x 512 space-time fine sweep (tv2d, configs 5 / 33)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_p.log 2>&1 || { tail gpurun_out/build_p.log; exit 1; }
timeout 300 python bench.py --config 4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p_c4.json 2>&1; echo "bench c4 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 9000 --csv --log-file gpurun_out/launches_c4_r2b.csv \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu launch c4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3r -s 3 -c 1 -o gpurun_out/ncu_tc3r_R5 \
  python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/ncu_tc3r_R5.log 2>&1; echo "ncu tc3r rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tv2d -s 3 -c 1 -o gpurun_out/ncu_tv2d_512 \
  python scripts/prof_op.py 2 0 2 512 512 tv > gpurun_out/ncu_tv2d_512.log 2>&1; echo "ncu tv2d rc=$?"
