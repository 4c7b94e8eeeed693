#!/bin/bash
# config-2 smoother knobs: nu (pre = post) x Jacobi weight cap
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "3 0.75" "2 0.75" "4 0.75" "3 0.85" "3 0.65" "2 0.85"; do set -- $v
  python bench.py --config ${CFG:-2} --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --nu $1 --omega $2 > gpurun_out/bs.json 2>gpurun_out/bs.err
  python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bs.json"))
    print("nu", sys.argv[1], "omega", sys.argv[2], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2), "ms its",
          d["solver"]["fwd_its"], d["solver"]["adj_its"])
except Exception:
    print("nu", sys.argv[1], "omega", sys.argv[2], "failed:", open("gpurun_out/bs.err").read().strip().splitlines()[-1][:160])
PY
done
