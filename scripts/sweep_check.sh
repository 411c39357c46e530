# quick sweep A/B on the box (not a bench value): C5 kernel times; PARITY=1 adds the sweep parity tests
mkdir -p gpurun_out
[ -n "$PARITY" ] && timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sweep or tile or fixture or random or c2_all or window" 2>&1 | tail -2
for w in ${WL:-c5}; do timeout 400 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-traffic --no-c4 > gpurun_out/$w.json 2>gpurun_out/$w.err; python -c "import json;d=json.load(open(\"gpurun_out/$w.json\"));print(\"$w\",d[\"value\"],d[\"e2e\"][\"value\"],{k:round(v,3) for k,v in d[\"kernel_ms\"].items()})"; done
