#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 33 5 4; do for cfg in "--nu-pre 2 --nu-post 2" "--nu-pre 1 --nu-post 2"; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline $cfg > gpurun_out/bnu.json 2>/dev/null
  python - "$c $cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/bnu.json")); s = d["solver"]
print("config", sys.argv[1], "|", round(d["value"]/1e6, 1), "MDOF/s", round(d["ms_per_step"]), "ms its", s["fwd_its"], s["adj_its"])
PY
done; done
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --nu-pre 1 --nu-post 2 --omega 0.8 > gpurun_out/bnu.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bnu.json')); s=d['solver']; print('config 3 (1,2) omega 0.8 |', round(d['value']/1e6,1), s['fwd_its'], s['adj_its'])"
