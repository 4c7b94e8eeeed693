#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e5.log 2>&1 || { tail gpurun_out/build_e5.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedules.py -q -k "preset or timestepping or fingerprint or null_adjoint" -p no:cacheprovider > gpurun_out/pytest_e5.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/pytest_e5.log | head -20
for c in 2 4; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --timestepping > gpurun_out/bts_c$c.json 2> gpurun_out/bts_c$c.err; echo "c$c rc=$?"; tail -3 gpurun_out/bts_c$c.err
python -c "import json; d=json.load(open('gpurun_out/bts_c$c.json')); print('config $c', round(d['value']/1e6,1), d['solver']['fwd_its'], d['timestepping'])"
done
