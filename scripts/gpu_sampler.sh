#!/bin/bash
# clock sampler started before the warm-up: config 2 / 4 / default benches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_m.log 2>&1 || { tail gpurun_out/build_m.log; exit 1; }
for c in 2 4; do
  timeout 900 python bench.py --config $c --timestepping > gpurun_out/bench_c${c}_m.json 2> gpurun_out/bench_c${c}_m.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py > gpurun_out/bench_default_m.json 2> gpurun_out/bench_default_m.err; echo "bench rc=$?"
timeout 900 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5_m.json 2> gpurun_out/bench_c5_m.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config 33 --no-cpu-baseline > gpurun_out/bench_c33_m.json 2> gpurun_out/bench_c33_m.err; echo "bench c33 rc=$?"
python scripts/results_table.py gpurun_out m
