cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out /tmp/ncu_reps
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ingest_pack -s 1 -c 1 -o /tmp/ncu_reps/ip -f python scripts/upload_kernels.py > gpurun_out/ip.log 2>&1
python scripts/ncu_summary.py /tmp/ncu_reps/ip.ncu-rep 60 > gpurun_out/ip_summary.txt 2>&1
python scripts/ncu_lines.py /tmp/ncu_reps/ip.ncu-rep 2000 > gpurun_out/ip_lines.txt 2>&1
