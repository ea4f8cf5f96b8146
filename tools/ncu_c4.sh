set -x
python tools/one_search.py C4 --target > gpurun_out/target.txt 2>&1 || exit 1
SKIP=$(grep -o "filter_skip [0-9]*" gpurun_out/target.txt | awk '{print $2}')
cat gpurun_out/target.txt
python tools/one_search.py C4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_filter -s $SKIP -c 1 -o gpurun_out/prof_c4_filter python tools/one_search.py C4 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
python tools/one_search.py C4 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 25000 --csv --log-file gpurun_out/launches_c4.csv python tools/one_search.py C4 > gpurun_out/ncu_list.log 2>&1
echo list rc=$?
ls -la gpurun_out/
