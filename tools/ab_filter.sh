for nt in 256 128 64; do
  for c in C4 C5 C3; do
    FT_FILTER_NT=$nt timeout 600 python bench.py --workload $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$c.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$c.json')); print('nt $nt $c', round(d['ms_per_step'],2), d['kernel_group_ms'])"
  done
done
