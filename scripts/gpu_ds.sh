#!/bin/bash
# st_design_step (fused forward + adjoint + sensitivities, overlapped host copies): its parity tests,
# the slab tests, and the benches of configs 2 and 3 (e2e through st_design_step)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "design_step or host_pointer" tests/test_gpu_slabs.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_ds_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ds_$TAG.log
for c in 2 3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/be_c$c.json 2> gpurun_out/be_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/be_c$c.json')); s=d['solver']; e=d['e2e']; print('config $c', round(d['value']/1e6,1), 'MDOF/s e2e', round(e['value']/1e6,1), e['ms_per_step'], 'ms', e['h2d_bytes_per_step'], e['d2h_bytes_per_step'], 'its', s['fwd_its'], s['adj_its'], 'clk', d['clocks']['sm_mhz'], d['clocks'].get('reasons'))" || tail -5 gpurun_out/be_c$c.err
done
