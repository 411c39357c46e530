#!/bin/bash
# Full ncu capture of one kernel, summarised on the box with the opcode mix:
# W=<workload> K=<kernel regex> S=<skip> TAG=<name> [EXTRA="bench args"]
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out /tmp/ncu_reps
rep=/tmp/ncu_reps/${TAG}
extra=""
[ "$W" = "c2" ] && extra="--no-c4"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${S:-1} -c 1 \
  -o $rep -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-traffic --workload $W $extra $EXTRA \
  > gpurun_out/${TAG}.log 2>&1
python scripts/ncu_summary.py $rep.ncu-rep 60 > gpurun_out/${TAG}_summary.txt 2>&1
python scripts/ncu_lines.py $rep.ncu-rep 2000 > gpurun_out/${TAG}_lines.txt 2>&1
python scripts/ncu_ops.py $rep.ncu-rep 60 > gpurun_out/${TAG}_ops.txt 2>&1
