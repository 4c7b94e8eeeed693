#!/bin/bash
# DGKS re-orthogonalisation threshold eta^2 (ST_DGKS_ETA2; 0 = never) vs iterations and time
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in 2 3 4; do for e in 0.5 0.01 0.0001 0; do
  ST_DGKS_ETA2=$e timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bd.json 2>gpurun_out/bd.err
  python - "$c" "$e" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bd.json")); s = d["solver"]
    print("config", sys.argv[1], "eta2", sys.argv[2], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 1), "ms its",
          s["fwd_its"], s["adj_its"], "rel_res", "%.2e" % s["rel_res"])
except Exception:
    print("config", sys.argv[1], "eta2", sys.argv[2], "failed:", open("gpurun_out/bd.err").read().strip().splitlines()[-1][:160])
PY
done; done
