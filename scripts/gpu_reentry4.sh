#!/bin/bash
# re-entry validation of HEAD (st_design_step state): GPU suite, smoke, default bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_default_$TAG.json')); print(round(d['value']/1e6,1), 'e2e', round(d['e2e']['value']/1e6,1), d['roofline']['frac'], d['clocks'])"
