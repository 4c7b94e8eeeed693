#!/bin/bash
# shared-memory V-cycle tail: parity subset, config-2 / config-3 A/B against per-level launches
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused or solve_adjoint or design" > gpurun_out/par_vt.log 2>&1; tail -2 gpurun_out/par_vt.log
for v in "1 2" "0 2" "1 3" "0 3"; do set -- $v
  ST_VTAIL=$1 python bench.py --config $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bvt.json 2>gpurun_out/bvt.err
  python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bvt.json"))
    print("vtail", sys.argv[1], "config", sys.argv[2], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2), "ms its",
          d["solver"]["fwd_its"], d["solver"]["adj_its"], "launches", d["gpu_launches"])
except Exception:
    print("vtail", sys.argv[1], "config", sys.argv[2], "failed:", open("gpurun_out/bvt.err").read().strip().splitlines()[-1][:200])
PY
done
