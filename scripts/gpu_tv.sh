#!/bin/bash
# tv2d iteration: parity (operator/coarse/variants/solve) + full-size certificate, kernel timings,
# plane-chunk A/B, ncu of the level-0/1 sweeps
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-tv}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/par_${TAG}.log 2>&1
tail -3 gpurun_out/par_${TAG}.log
{
for lv in 0 1; do echo -n "256^3 tv level $lv JAC: "; python scripts/prof_op.py 2 $lv 2 256 256 tv 2>&1 | tail -1; done
for lv in 0 1; do echo -n "512^2x512 tv level $lv JAC: "; python scripts/prof_op.py 2 $lv 2 512 512 tv 2>&1 | tail -1; done
for mb in 16 48; do for lv in 0 1; do echo -n "ST_CHUNK_MB=$mb 512^2x512 tv level $lv JAC: "; ST_CHUNK_MB=$mb python scripts/prof_op.py 2 $lv 2 512 512 tv 2>&1 | tail -1; done; done
} > gpurun_out/kb_${TAG}.log 2>&1
cat gpurun_out/kb_${TAG}.log
if [ -n "$PROF" ]; then TAG=$TAG bash scripts/gpu_prof_tv.sh; fi
