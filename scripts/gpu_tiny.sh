#!/bin/bash
# one-thread-per-node kernel for small time-constant levels: parity subset, threshold A/B on config 2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "coarse or variants or solve_adjoint or fused or prolongation or design" > gpurun_out/par_tiny.log 2>&1; tail -1 gpurun_out/par_tiny.log
for tn in 0 20000 300000 1100000 4300000; do
  ST_TINY_NODES=$tn timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bt.json 2>gpurun_out/bt.err
  python - "$tn" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/bt.json")); s = d["solver"]
    print("tiny<=", sys.argv[1], round(d["value"] / 1e6, 1), "MDOF/s", round(d["ms_per_step"], 2), "ms its", s["fwd_its"], "setup", s["setup_ms"][:2])
except Exception:
    print("tiny<=", sys.argv[1], "failed:", open("gpurun_out/bt.err").read().strip().splitlines()[-1][:160])
PY
done
