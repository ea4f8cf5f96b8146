# usage: bash tools/ncu_kernels.sh  -> full-set captures of the hot kernels
set -x
python tools/one_search.py C4 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_filter -s 60 -c 1 -o gpurun_out/prof_c4_filter2 python tools/one_search.py C4 > gpurun_out/ncu_a.log 2>&1
echo a=$?
ncu --set full --clock-control none --import-source on -k regex:k_bucket_large -s 60 -c 1 -o gpurun_out/prof_c4_bucket python tools/one_search.py C4 > gpurun_out/ncu_b.log 2>&1
echo b=$?
python tools/one_search.py C5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_direct -s 12 -c 1 -o gpurun_out/prof_c5_direct python tools/one_search.py C5 > gpurun_out/ncu_c.log 2>&1
echo c=$?
