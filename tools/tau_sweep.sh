N=$1; shift
for tau in "$@"; do
  for c in C4 C5; do
    FT_REPLICATE_TAU=$tau timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --workload $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tau_$c.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/tau_$c.json')); print('N=$N tau=$tau $c', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), d['kernel_group_ms'])"
  done
done
