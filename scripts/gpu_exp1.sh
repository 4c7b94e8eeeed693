#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e1.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "solve_adjoint or prolongation or coarse_operators or config2 or config3-shaped-256" -p no:cacheprovider > gpurun_out/pytest_e1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_e1.log
for nf in 0 50000000 200000000; do
  timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --nu-fine-nodes $nf > gpurun_out/b3_nf$nf.json 2> gpurun_out/b3_nf$nf.err
  python - "$nf" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/b3_nf{sys.argv[1]}.json").read())
print("nu_fine_nodes", sys.argv[1], round(d["value"]/1e6, 1), "MDOF/s", round(d["ms_per_step"]), "ms its", d["solver"]["fwd_its"], d["solver"]["adj_its"], "setup", d["solver"]["setup_ms"], "sweep us", round(d["roofline"]["us_per_launch"]))
PY
done
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b2_e1.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/b2_e1.json')); print('config2', round(d['value']/1e6,1), d['ms_per_step'], d['solver']['fwd_its'], d['solver']['adj_its'])"
python scripts/prof_op.py 2 0 2 1024 1024 tv > gpurun_out/profop_c3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:tv2d_kernel -s 3 -c 1 -o gpurun_out/ncu_tv2d_c3 python scripts/prof_op.py 2 0 2 1024 1024 tv > gpurun_out/ncu_tv2d_c3.log 2>&1; echo ncu rc=$?; cat gpurun_out/profop_c3.log
