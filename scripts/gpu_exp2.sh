#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e2.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_schedules.py -q -x -k "tv2d" -p no:cacheprovider > gpurun_out/pytest_e2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_e2.log
for k in 16 32 64 128 -1; do python scripts/prof_op.py 2 0 2 1024 1024 tv chunk_planes=$k; done 2>&1 | tee gpurun_out/kbench_c3_chunk.log
for k in 16 64 -1; do python scripts/prof_op.py 2 0 2 512 512 tv chunk_planes=$k; python scripts/prof_op.py 2 1 2 1024 1024 tv chunk_planes=$k; done 2>&1 | tee -a gpurun_out/kbench_c3_chunk.log
for k in 32 -1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tv2d_kernel -s 3 -c 1 python scripts/prof_op.py 2 0 2 1024 1024 tv chunk_planes=$k > gpurun_out/ncu_dram_k$k.log 2>&1
  echo "K=$k"; grep -E "dram__bytes|duration|hit_rate" gpurun_out/ncu_dram_k$k.log
done
