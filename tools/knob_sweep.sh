# A/B of the sampling / capacity knobs on C5 and C4: one bench
# line per setting -> gpurun_out/sweep_<W>_<setting>.json
for W in C5 C4; do
  for KV in "BASE=1" "FT_SLOG=3" "FT_SLOG=5" "FT_SLOG0=3" "FT_SLOG0=1" "FT_CDIRECT=2048" "FT_SMALL_WAVE=0" "FT_SMALL_WAVE=65536" "FT_ITEM_MAX=256" "FT_ITEM_MAX=1024"; do
    env $KV python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sweep_${W}_${KV}.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${W}_${KV}.json')); print('$W', '$KV', round(d['ms_per_step'],2), d['kernel_group_ms'])"
  done
done
