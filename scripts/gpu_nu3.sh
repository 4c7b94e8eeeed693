#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "--nu-pre 1 --nu-post 2" "--nu-pre 1 --nu-post 3" "--nu-pre 2 --nu-post 1" "--nu-pre 1 --nu-post 2 --nu-coarse 4" "--nu-coarse 4"; do
  timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline $cfg > gpurun_out/bnu.json 2>/dev/null
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/bnu.json")); s = d["solver"]
print(sys.argv[1], "|", round(d["value"]/1e6, 1), "MDOF/s", round(d["ms_per_step"]), "ms its", s["fwd_its"], s["adj_its"], "vc", s["fwd_vcycles"])
PY
done
