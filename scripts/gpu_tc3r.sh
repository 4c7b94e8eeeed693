#!/bin/bash
# tc3r (element-layer (3+1)D fine-level kernel) A/B: parity on the 3D cases, then config-4 level-0
# kernel times for R = 2, R = 4 and the tc3d stencil kernel, then config-4 bench with the default
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B=paper_2508_09589_b200
variant() {  # $1 = extra nvcc flags
  rm -f $B/build/tc3r.o
  ST_NVCC_EXTRA="$1" python -c "from paper_2508_09589_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build failed: $1"
}
variant ""
timeout 1200 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py "tests/test_gpu_fullsize.py::test_fullsize_solution_certified_by_oracle_rows[config4]" -m gpu -q -x -p no:cacheprovider > gpurun_out/t3r_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t3r_pytest.log
for v in "-DST_TC3R_R=2" "-DST_TC3R_R=4" "-DST_TC3R_OFF"; do
  variant "$v"
  for m in 2 1 0 3; do echo -n "$v mode $m: "; timeout 300 python scripts/prof_op.py $m 0 3 64 128 tc c4 2>&1 | tail -1; done
done > gpurun_out/t3r_kbench.log 2>&1
cat gpurun_out/t3r_kbench.log
variant ""
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/t3r_bench_c4.json 2> gpurun_out/t3r_bench_c4.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/t3r_bench_c4.json')); s=d['solver']; print('config 4', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'], 'roof', d.get('roofline'))"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mdot_bench scripts/dev/mdot_bench.cu && timeout 300 /tmp/mdot_bench > gpurun_out/mdot_bench.log 2>&1; cat gpurun_out/mdot_bench.log
