#!/bin/bash
# ncu capture of one kernel: KERNEL=<regex> [TAG=name]
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
K=${KERNEL:-k_sweep}
T=${TAG:-$K}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
   -o gpurun_out/prof_$T -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 > gpurun_out/ncu_$T.log 2>&1
tail -3 gpurun_out/ncu_$T.log
