#!/bin/bash
# fine-level sweeps (--nu) x coarse-level sweeps (ST_NU_COARSE)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in 2 3; do for v in "4 4" "3 4" "4 3" "3 5" "4 2" "5 3" "4 5"; do set -- $v
  ST_NU_COARSE=$2 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --nu $1 > gpurun_out/bn.json 2>gpurun_out/bn.err
  python - "$c" "$1" "$2" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bn.json")); s = d["solver"]
    print("config", sys.argv[1], "fine", sys.argv[2], "coarse", sys.argv[3], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2),
          "ms its", s["fwd_its"], s["adj_its"])
except Exception:
    print("config", sys.argv[1], "fine", sys.argv[2], "coarse", sys.argv[3], "failed:", open("gpurun_out/bn.err").read().strip().splitlines()[-1][:160])
PY
done; done
