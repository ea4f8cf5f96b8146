# Round evidence (single GPU): bench lines, launch list of the bench command,
# full-set captures of the top kernels at their largest launch.
set -x
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?
python bench.py --workload C5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20000 --csv \
    --log-file gpurun_out/launches_c4_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
echo list rc=$?
cap() {  # workload target-kernel out [wave]
  if [ -n "$4" ]; then python tools/one_search.py $1 --target $2 --wave $4 > gpurun_out/target_$3.txt 2>&1 || return 1
  else python tools/one_search.py $1 --target $2 > gpurun_out/target_$3.txt 2>&1 || return 1; fi
  SKIP=$(grep -o "skip [0-9]*" gpurun_out/target_$3.txt | awk '{print $2}')
  ncu --set full --clock-control none --import-source on -k regex:"^$2\$|$2\(" -s $SKIP -c 1 -o gpurun_out/$3 python tools/one_search.py $1 > gpurun_out/ncu_$3.log 2>&1
  echo "$3 rc=$?"
}
cap C4 k_filter r1_c4_k_filter
cap C5 k_filter r1_c5_k_filter
cap C4 k_bucket_small r1_c4_k_bucket_small
cap C5 k_node_pack r1_c5_k_node_pack 1
cap C4 k_direct r1_c4_k_direct 4
