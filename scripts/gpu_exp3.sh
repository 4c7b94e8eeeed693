#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e3.log 2>&1 || exit 1
for lv in 0 1 2; do for k in 0 -1 64; do python scripts/prof_op.py 2 $lv 2 1024 1024 tv chunk_planes=$k; done; done 2>&1 | tee gpurun_out/kbench_c3_g.log
for lv in 0 1; do for k in 0 -1 32 64; do python scripts/prof_op.py 2 $lv 2 512 512 tv chunk_planes=$k; done; done 2>&1 | tee -a gpurun_out/kbench_c3_g.log
for nf in 50000000 10000000; do
  timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --nu-fine-nodes $nf > gpurun_out/b3g_nf$nf.json 2> gpurun_out/b3g_nf$nf.err
  python - "$nf" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/b3g_nf{sys.argv[1]}.json").read())
print("nu_fine_nodes", sys.argv[1], round(d["value"]/1e6, 1), "MDOF/s", round(d["ms_per_step"]), "ms its", d["solver"]["fwd_its"], d["solver"]["adj_its"], "sweep us", round(d["roofline"]["us_per_launch"]), "frac", round(d["roofline"]["frac"], 3), round(d["roofline"]["min_frac"], 3), "step frac", round(d["step_roofline"]["frac"], 3))
PY
done
for c in 33 5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --nu-fine-nodes 50000000 > gpurun_out/bg_c$c.json 2> gpurun_out/bg_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bg_c$c.json')); print('config $c nf5e7', round(d['value']/1e6,1), round(d['ms_per_step'],1), d['solver']['fwd_its'], d['solver']['adj_its'])"
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --nu-fine-nodes 0 > gpurun_out/bg0_c$c.json 2> gpurun_out/bg0_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bg0_c$c.json')); print('config $c nf0', round(d['value']/1e6,1), round(d['ms_per_step'],1), d['solver']['fwd_its'], d['solver']['adj_its'])"
done
