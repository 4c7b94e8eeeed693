#!/bin/bash
# config-2 solve with the paper's preconditioner variants (GMRES(10)-Jacobi smoother, full coarsening)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
i=0
for a in "--smoother gmres" "--smoother gmres --full-coarsening" "--full-coarsening"; do
  i=$((i+1))
  timeout 900 python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 $a > gpurun_out/pv$i.json 2> gpurun_out/pv$i.err
  python - "$a" gpurun_out/pv$i.json gpurun_out/pv$i.err <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2])); s = d["solver"]
    print(sys.argv[1], "|", d["config"]["preconditioner"], "|", round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 1),
          "ms/step; its fwd", s["fwd_its"], "adj", s["adj_its"])
except Exception:
    print(sys.argv[1], "| failed:", open(sys.argv[3]).read().strip().splitlines()[-1][:200])
PY
done
