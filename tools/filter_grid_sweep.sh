# k_filter grid / register-budget A/B on C5 and C4
for W in C5 C4; do
  for KV in "BASE=1" "FT_FILTER_GRID=888" "FT_FILTER_GRID=1776" "FT_FILTER_GRID=4736" "FT_FILTER_GRID=9472" "FT_FILTER_GRID=75776" "FT_FILTER_REGS=64 FT_FILTER_GRID=1184" "FT_FILTER_REGS=64 FT_FILTER_GRID=4736"; do
    env $KV python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/fg.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/fg.json')); print('$W', '$KV', round(d['ms_per_step'],2), d['kernel_group_ms'])"
  done
done
