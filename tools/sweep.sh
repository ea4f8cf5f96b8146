timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py --timeout 800 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gpu_tests.log
for c in C4 C5 C3; do
  timeout 600 python bench.py --workload $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>/dev/null; python -c "import json,sys; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']/1e9,2), round(d['ms_per_step'],2), d['kernel_group_ms'], round(d['e2e']['ms_per_step'],2), d['gpu_launches'], d['ft_steps'], d['roofline']['kernel'], round(d['roofline']['frac'] or 0,3))"
done
