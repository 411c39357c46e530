#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full captures.
set -x
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 1 -c 1 \
     -o gpurun_out/prof_sim -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 > gpurun_out/ncu_sim.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 \
     -o gpurun_out/prof_sweep -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 > gpurun_out/ncu_sweep.log 2>&1
fi
ls -la gpurun_out
