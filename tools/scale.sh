N=$1
for c in C4 C5; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N tools/dist_check.py $c > gpurun_out/dist${N}_$c.log 2>&1; echo dist $c rc=$?; grep -E "^rank 0" gpurun_out/dist${N}_$c.log | head -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --workload $c --steps 5 --warmup 3 > gpurun_out/bench${N}_$c.json 2>gpurun_out/bench${N}_$c.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench${N}_$c.json')); print('$c N=$N', round(d['value']/1e9,2), 'Gt/s', round(d['ms_per_step'],2), 'ms', d['kernel_group_ms'], 'e2e', round(d['e2e']['ms_per_step'],2))"
done
