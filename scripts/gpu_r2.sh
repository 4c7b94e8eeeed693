#!/bin/bash
# round-2 GPU validation: build, GPU tests, benches (usage: scripts/gpu_r2.sh TAG [pytest-args...])
TAG=${1:-a}; shift
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --durations=30 "$@" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
