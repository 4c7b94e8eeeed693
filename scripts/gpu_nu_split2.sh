#!/bin/bash
# second round: fine-level sweeps (--nu) x coarse-level sweeps (ST_NU_COARSE), all configs
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
run() {
  ST_NU_COARSE=$3 timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --nu $2 > gpurun_out/bn.json 2>gpurun_out/bn.err
  python - "$1" "$2" "$3" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bn.json")); s = d["solver"]
    print("config", sys.argv[1], "fine", sys.argv[2], "coarse", sys.argv[3], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2),
          "ms its", s["fwd_its"], s["adj_its"])
except Exception:
    print("config", sys.argv[1], "fine", sys.argv[2], "coarse", sys.argv[3], "failed:", open("gpurun_out/bn.err").read().strip().splitlines()[-1][:160])
PY
}
for v in "2 5" "2 6" "3 6" "2 8"; do run 2 $v; done
for v in "2 4" "2 5" "3 6"; do run 3 $v; done
for v in "4 4" "3 4" "3 5" "2 5" "3 6"; do run 4 $v; done
for v in "4 4" "3 4" "3 5" "2 5"; do run 5 $v; done
