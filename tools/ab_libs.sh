# A/B of prebuilt libft variants in abl/: python bench per variant (C4, C5)
cp paper_2004_10856_b200/libft.so /tmp/libft_orig.so
for v in "$@"; do
  cp abl/libft_$v.so paper_2004_10856_b200/libft.so
  for c in C4 C5; do
    timeout 600 python bench.py --workload $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$c.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$c.json')); print('$v $c', round(d['ms_per_step'],2), d['kernel_group_ms'])"
  done
done
cp /tmp/libft_orig.so paper_2004_10856_b200/libft.so
