#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in 2 3 5; do for f in 1.5 1.8 1.95; do
  ST_OMEGA_FAC=$f timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bo.json 2>gpurun_out/bo.err
  python -c "import json; d=json.load(open('gpurun_out/bo.json')); s=d['solver']; print('config $c fac $f', round(d['value']/1e6,1), 'MDOF/s its', s['fwd_its'], s['adj_its'])" 2>/dev/null || echo "config $c fac $f failed: $(tail -1 gpurun_out/bo.err | cut -c1-150)"
done; done
