for cfg in "FT_WARP16=1" "FT_WARP16=0"; do for c in C4 C5 C3; do
  env $cfg timeout 600 python bench.py --workload $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $cfg', round(d['value']/1e9,2), round(d['ms_per_step'],2), d['kernel_group_ms'], d['gpu_launches']//5)"
done; done
