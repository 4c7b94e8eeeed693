#!/bin/bash
# end-of-round validation: GPU tests, smoke, benches (configs 2-5), launch list + ncu of the dominant kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-final}
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/par_$TAG.log 2>&1; tail -1 gpurun_out/par_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err; echo "bench rc=$?"
for c in 3 4 5; do python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c$c.json 2>>gpurun_out/bench_$TAG.err; done
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_${TAG}_ref.json 2>>gpurun_out/bench_$TAG.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc2d -s 3 -c 1 -o gpurun_out/prof_tc2d_$TAG \
  python scripts/prof_op.py 2 0 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
