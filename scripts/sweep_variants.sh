mkdir -p gpurun_out
for S in 64 32; do for v in 0 1 2; do
  TBSIM_SWEEP_S=$S TBSIM_SWEEP_VARIANT=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-c4 2>&1 | tail -1 | python scripts/summ.py c2S${S}v$v
done; done
