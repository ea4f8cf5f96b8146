for W in C5 C4; do
  for KV in "BASE=1" "FT_PACK_GRID=444" "FT_PACK_GRID=296" "FT_PACK_GRID=888" "FT_PACK_GRID=1184"; do
    env $KV python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/pg.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/pg.json')); print('$W', '$KV', round(d['ms_per_step'],2), d['kernel_group_ms'])"
  done
done
