# Round-1 ncu evidence (single GPU).  1) launch list of the bench command,
# 2) full-set captures of the dominant kernels at their largest launch.
set -x
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16000 --csv \
    --log-file gpurun_out/launches_c4_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
echo list rc=$?
cap() {  # workload kernel-family target-kernel out
  python tools/one_search.py $1 --target $2 > gpurun_out/target_$4.txt 2>&1 || return 1
  SKIP=$(grep -o "skip [0-9]*" gpurun_out/target_$4.txt | awk '{print $2}')
  ncu --set full --clock-control none --import-source on -k regex:"$3" -s $SKIP -c 1 -o gpurun_out/$4 python tools/one_search.py $1 > gpurun_out/ncu_$4.log 2>&1
  echo "$4 rc=$?"
}
python tools/one_search.py C4 > gpurun_out/plain_c4.log 2>&1 && cap C4 k_filter k_filter r1_c4_k_filter
cap C4 k_bucket_small k_bucket_small r1_c4_k_bucket_small
python tools/one_search.py C5 > gpurun_out/plain_c5.log 2>&1 && cap C5 k_filter k_filter r1_c5_k_filter
