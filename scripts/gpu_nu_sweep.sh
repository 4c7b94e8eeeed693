#!/bin/bash
# smoothing-sweep count per config (pre = post)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "2 5" "2 6" "3 5" "4 3" "4 4" "5 3" "5 4"; do set -- $v
  timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --nu $2 > gpurun_out/bs.json 2>gpurun_out/bs.err
  python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bs.json"))
    print("config", sys.argv[1], "nu", sys.argv[2], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2), "ms its",
          d["solver"]["fwd_its"], d["solver"]["adj_its"])
except Exception:
    print("config", sys.argv[1], "nu", sys.argv[2], "failed:", open("gpurun_out/bs.err").read().strip().splitlines()[-1][:160])
PY
done
