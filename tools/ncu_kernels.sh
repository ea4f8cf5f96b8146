# full-set ncu captures of the hot kernels at their biggest launch
set -x
cap() {  # workload kernel out
  python tools/one_search.py $1 --target $2 > gpurun_out/target_$3.txt 2>&1 || return 1
  SKIP=$(grep -o "skip [0-9]*" gpurun_out/target_$3.txt | awk '{print $2}')
  ncu --set full --clock-control none --import-source on -k regex:"^$2\b|$2\(" -s $SKIP -c 1 -o gpurun_out/$3 python tools/one_search.py $1 > gpurun_out/ncu_$3.log 2>&1
  echo "$3 rc=$?"
}
python tools/one_search.py C4 > gpurun_out/plain_c4.log 2>&1 && cap C4 k_filter prof_c4_filter
python tools/one_search.py C5 > gpurun_out/plain_c5.log 2>&1 && cap C5 k_direct_warp prof_c5_dwarp
cap C4 k_bucket_small prof_c4_bsmall
