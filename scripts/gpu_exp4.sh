#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e4.log 2>&1 || exit 1
for rep in 1 2; do for c in 0 -1; do python scripts/prof_op.py 2 0 2 1024 1024 tv max_ctas=$c; python scripts/prof_op.py 2 0 2 512 512 tv max_ctas=$c; done; done 2>&1 | tee gpurun_out/kbench_trim.log
python scripts/prof_op.py 2 1 2 512 512 tv 2>&1 | tee -a gpurun_out/kbench_trim.log
for c in 33 5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --nu-fine-nodes 10000000 > gpurun_out/bh_c$c.json 2> gpurun_out/bh_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bh_c$c.json')); print('config $c nf1e7', round(d['value']/1e6,1), round(d['ms_per_step'],1), d['solver']['fwd_its'], d['solver']['adj_its'])"
done
timeout 900 python bench.py --config 3 --nu-fine-nodes 10000000 > gpurun_out/bench_c3_full.json 2> gpurun_out/bench_c3_full.err; echo "c3 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3_full.json')); print('config 3 full', round(d['value']/1e6,1), round(d['ms_per_step'],1), d['solver']['fwd_its'], d['solver']['adj_its'], 'e2e', round(d['e2e']['value']/1e6,1), 'cpu', d['cpu_baseline']['value'], 'mem', d['solver']['device_mem_used_gb'], d['clocks'])"
