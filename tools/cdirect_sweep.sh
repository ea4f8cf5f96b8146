# direct-capacity A/B: global FT_CDIRECT and the small-wave threshold FT_SMALL_WAVE
for cfg in "FT_SMALL_WAVE=0" "FT_SMALL_WAVE=1024" "FT_SMALL_WAVE=4096"; do for c in C4 C5 C3; do
env $cfg timeout 600 python bench.py --workload $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg $c', round(d['ms_per_step'],2), d['kernel_group_ms'])"
done; done
