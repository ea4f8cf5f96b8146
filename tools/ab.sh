timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py --timeout 800 2>&1 | tail -1
for c in C4 C5 C3; do
  timeout 600 python bench.py --workload $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']/1e9,2), round(d['ms_per_step'],2), d['kernel_group_ms'], d['gpu_launches']//3)"
done
python tools/waves.py C4 > gpurun_out/w1.txt; head -5 gpurun_out/w1.txt
