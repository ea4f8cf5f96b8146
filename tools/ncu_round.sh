# Round-2 evidence on one GPU (run from the repo root under gpurun; outputs
# in gpurun_out/): per-kernel counters of one search (C5, C4) ->
# r2_kernels.json (copied to profiles/ so the bench roofline reads it), the
# bench lines (after the JSON is in place), the launch list of the bench
# command and a --set full capture of the largest k_filter launch.
set -x
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
rm -f gpurun_out/r2_kernels.json
for W in C5 C4; do
  ncu --metrics $M --clock-control none -c 40000 --csv --log-file gpurun_out/r2_launches_$W.csv \
      python tools/one_search.py $W > gpurun_out/r2_ncu_list_$W.log 2>&1
  echo list $W rc=$?
  python tools/kernel_table.py gpurun_out/r2_launches_$W.csv $W --out gpurun_out/r2_kernels.json > gpurun_out/r2_kernels_$W.txt
done
cp gpurun_out/r2_kernels.json profiles/r2_kernels.json
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo bench rc=$?
python bench.py --workload C4 --no-cpu-baseline > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
for W in C2 C3; do python bench.py --workload $W --no-cpu-baseline > gpurun_out/r2_bench_$W.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/r2_bench_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2_ncu_bench.log 2>&1
echo bench-list rc=$?
python tools/one_search.py C5 --target k_filter > gpurun_out/r2_target.txt 2>&1
SKIP=$(grep -o "skip [0-9]*" gpurun_out/r2_target.txt | awk '{print $2}')
ncu --set full --clock-control none --import-source on -k regex:k_filter -s $SKIP -c 1 \
    -o gpurun_out/r2_c5_k_filter python tools/one_search.py C5 > gpurun_out/r2_ncu_full.log 2>&1
echo full rc=$?
