#!/bin/bash
# re-entry validation of HEAD: GPU suite, smoke, default bench (config 3), configs 2 and 4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-v}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
for c in 2 4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_c${c}_$TAG.json 2> gpurun_out/bench_c${c}_$TAG.err; echo "bench c$c rc=$?"
done
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
for f in ["default", "c2", "c4"]:
    try:
        d = json.load(open(f"gpurun_out/bench_{f}_{t}.json"))
    except Exception as e:
        print(f, "failed", e); continue
    r = d.get("roofline") or {}
    print(f, round(d["value"] / 1e6, 2), "MDOF/s", round(d["ms_per_step"], 1), "ms", "e2e", round((d.get("e2e") or {}).get("value", 0) / 1e6, 1),
          "frac", round(r.get("frac", 0), 3), "minfrac", round(r.get("min_frac", 0), 3), "step", round((d.get("step_roofline") or {}).get("frac", 0), 3),
          "its", (d.get("solver") or {}).get("fwd_its"), (d.get("solver") or {}).get("adj_its"), "clk", (d.get("clocks") or {}).get("sm_mhz"),
          (d.get("clocks") or {}).get("reasons"))
PY
