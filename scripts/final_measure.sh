#!/bin/bash
# Every bench line of this build on one box: C2 (the driver's default run),
# the reference arm, C1, C3, C4 (with the reference cpu_baseline and
# config-scale parity), C5; then the ncu launch list of the C2 step.
# TAG=<name> prefixes the outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
T=${TAG:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${T}_gpu.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
for w in c1 c3 c5; do
  timeout 900 python bench.py --workload $w > gpurun_out/${T}_$w.json 2> gpurun_out/${T}_$w.err
done
timeout 1200 python bench.py --workload c4 --steps 3 --warmup 1 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
   --log-file gpurun_out/${T}_c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --no-traffic > /dev/null 2>&1
ls -la gpurun_out | grep ${T}_
