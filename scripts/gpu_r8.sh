#!/bin/bash
# restart length on the 512^2x512 workloads (config-3 slab, config 5)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_n.log 2>&1 || { tail gpurun_out/build_n.log; exit 1; }
run() { local c=$1 lab=$2; shift 2
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 3 "$@" > gpurun_out/bn_$lab.json 2> gpurun_out/bn_$lab.err
  python -c "import json; d=json.load(open('gpurun_out/bn_$lab.json')); s=d['solver']; print('c$c $lab', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bn_$lab.err
}
run 33 c33base
run 33 c33r8 --restart 8
run 33 c33r10 --restart 10
run 5 c5base
run 5 c5r8 --restart 8
run 5 c5r10 --restart 10
