"""Markdown rows of DESIGN.md sec. 10 / README from bench JSON lines: results_table.py DIR TAG"""
import json, sys, os
d, tag = sys.argv[1], sys.argv[2]
names = [("default", "config 3"), ("c2", "config 2"), ("c33", "config 3 slab 512^2x512"), ("c4", "config 4"), ("c5", "config 5")]
for f, lab in names:
    p = os.path.join(d, f"bench_{f}_{tag}.json")
    if not os.path.exists(p):
        continue
    j = json.load(open(p))
    r, s, e, sr = j.get("roofline") or {}, j.get("solver") or {}, j.get("e2e") or {}, j.get("step_roofline") or {}
    fi, ai = s.get("fwd_its") or [0], s.get("adj_its") or [0]
    ts = (j.get("timestepping") or {}).get("space_time_speedup_forward")
    print(f"| {lab} | {j['value']/1e6:.1f} | {j['ms_per_step']:.1f} | {e.get('value', 0)/1e6:.1f} | "
          f"{min(fi)}-{max(fi)} / {min(ai)}-{max(ai)} | {r.get('frac', 0):.3f} / {r.get('min_frac', 0):.3f} "
          f"({r.get('us_per_launch', 0):.0f} us) | {sr.get('frac', 0):.3f} | clk {j['clocks']['sm_mhz']} {j['clocks'].get('reasons')} "
          f"| launches {j.get('gpu_launches')} | ts {ts}")
