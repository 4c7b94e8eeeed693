#!/bin/bash
# CUDA-graph coverage of the V-cycle: levels below ST_GRAPH_NODES nodes (default 2^19)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in 2 3; do for gn in 524288 8388608 1073741824; do
  ST_GRAPH_NODES=$gn timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bg.json 2>gpurun_out/bg.err
  python - "$c" "$gn" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bg.json")); s = d["solver"]
    print("config", sys.argv[1], "graph<", sys.argv[2], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2), "ms its", s["fwd_its"])
except Exception:
    print("config", sys.argv[1], "graph<", sys.argv[2], "failed:", open("gpurun_out/bg.err").read().strip().splitlines()[-1][:160])
PY
done; done
