#!/bin/bash
# FGMRES(8) on the 512^2x512 bench workloads: full-size certification and the bench lines
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_o.log 2>&1 || { tail gpurun_out/build_o.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "not config3_fullsize" > gpurun_out/pytest_o.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_o.log
timeout 900 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5_o.json 2> gpurun_out/bench_c5_o.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config 33 --no-cpu-baseline > gpurun_out/bench_c33_o.json 2> gpurun_out/bench_c33_o.err; echo "bench c33 rc=$?"
python scripts/results_table.py gpurun_out o
