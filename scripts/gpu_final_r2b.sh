#!/bin/bash
# round-2 final evidence (second pass, after the transfer kernels / st_design_step): GPU suite, smoke, every bench workload, reference arm, the launch list of the
# default bench command, ncu --set full of its dominant kernel (config-3 fine-level sweep)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"
for c in 2 4 5 33; do
  extra=""; if [ $c = 2 ] || [ $c = 4 ]; then extra="--timestepping"; fi
  timeout 900 python bench.py --config $c $extra > gpurun_out/bench_c${c}_$TAG.json 2> gpurun_out/bench_c${c}_$TAG.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
for f in ["default", "c2", "c4", "c5", "c33", "ref"]:
    try:
        d = json.load(open(f"gpurun_out/bench_{f}_{t}.json"))
    except Exception as e:
        print(f, "failed", e); continue
    r = d.get("roofline") or {}
    print(f, round(d["value"] / 1e6, 2), "MDOF/s", round(d["ms_per_step"], 1), "ms", "e2e", round((d.get("e2e") or {}).get("value", 0) / 1e6, 1),
          "frac", round(r.get("frac", 0), 3), "minfrac", round(r.get("min_frac", 0), 3), "step", round((d.get("step_roofline") or {}).get("frac", 0), 3),
          "its", (d.get("solver") or {}).get("fwd_its"), (d.get("solver") or {}).get("adj_its"), "clk", (d.get("clocks") or {}).get("sm_mhz"),
          (d.get("clocks") or {}).get("reasons"), "ts", (d.get("timestepping") or {}).get("space_time_speedup_forward"))
PY
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c3_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c3_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tv2d_kernel -s 3 -c 1 -o gpurun_out/ncu_tv2d_c3_$TAG \
  python scripts/prof_op.py 2 0 2 1024 1024 tv > gpurun_out/ncu_tv2d_c3_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/launches_c2_$TAG.csv \
  python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_c2_$TAG.log 2>&1; echo "ncu launch c2 rc=$?"
for c in 2 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 3 --restart 6 > gpurun_out/bench_c${c}_r6_$TAG.json 2> gpurun_out/bench_c${c}_r6_$TAG.err
  python -c "import json; d=json.load(open('gpurun_out/bench_c${c}_r6_$TAG.json')); s=d['solver']; print('c$c restart 6', round(d['value']/1e6,1), 'MDOF/s', round(d['ms_per_step'],1), 'ms its', s['fwd_its'], s['adj_its'])"
done
