#!/bin/bash
# tc3r R = 2 / R = 4: kernel times and one ncu --set full capture of the config-4 fine JAC sweep each
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B=paper_2508_09589_b200
variant() { rm -f $B/build/tc3r.o; ST_NVCC_EXTRA="$1" python -c "from paper_2508_09589_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build failed: $1"; }
for R in 2 4; do
  variant "-DST_TC3R_R=$R"
  for m in 2 1 3; do echo -n "R=$R mode $m: "; timeout 300 python scripts/prof_op.py $m 0 3 64 128 tc c4 2>&1 | tail -1; done
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3r -s 3 -c 1 -o gpurun_out/ncu_tc3r_R$R \
     python scripts/prof_op.py 2 0 3 64 128 tc c4 > gpurun_out/ncu_tc3r_R$R.log 2>&1; echo "ncu R=$R rc=$?"
done
