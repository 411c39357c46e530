#!/bin/bash
# One profiling session (ncu; never a bench value): per-launch DRAM bytes +
# duration of every kernel for C2 and C4, full captures of the top kernels,
# summarised ON THE BOX (the .ncu-rep files stay there unless KEEP_REP=1;
# gpurun brings back <= 64 MiB).  TAG=<name> names the outputs.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out /tmp/ncu_reps
T=${TAG:-prof}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-traffic"
if [ -z "$SKIP_LAUNCHES" ]; then
  timeout 900 ncu --metrics $M --clock-control none -c 120 --csv --log-file gpurun_out/${T}_c2_launches.csv $B --no-c4 > /dev/null 2>&1
  timeout 900 ncu --metrics $M --clock-control none -c 60 --csv --log-file gpurun_out/${T}_c4_launches.csv $B --workload c4 > /dev/null 2>&1
fi
full() {  # full <workload> <kernel regex> <skip>
  local w=$1 k=$2 s=${3:-1} extra=""
  [ "$w" = "c2" ] && extra="--no-c4"
  local rep=/tmp/ncu_reps/${T}_${w}_$k
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
    -o $rep -f $B --workload $w $extra > gpurun_out/${T}_${w}_$k.log 2>&1
  python scripts/ncu_summary.py $rep.ncu-rep 40 > gpurun_out/${T}_${w}_${k}_summary.txt 2>&1
  python scripts/ncu_lines.py $rep.ncu-rep 60 > gpurun_out/${T}_${w}_${k}_lines.txt 2>&1
  [ -n "$KEEP_REP" ] && cp $rep.ncu-rep gpurun_out/
}
for k in $FULL_C1; do full c1 $k 1; done
for k in $FULL_C2; do full c2 $k 1; done
for k in $FULL_C3; do full c3 $k 1; done
for k in $FULL_C4; do full c4 $k 1; done
ls -la gpurun_out | tail -30
