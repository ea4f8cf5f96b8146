python tools/one_search.py C4 > gpurun_out/plain_c4.log 2>&1
for k in k_direct_warp16 k_direct_warp; do
python tools/one_search.py C4 --target $k --wave 2 > gpurun_out/t_$k.txt 2>&1
SKIP=$(grep -o "skip [0-9]*" gpurun_out/t_$k.txt | awk '{print $2}')
ncu --set full --clock-control none --import-source on -k regex:"^$k\$|$k\(" -s $SKIP -c 1 -o gpurun_out/w2_$k python tools/one_search.py C4 > gpurun_out/ncu_w2_$k.log 2>&1; echo $k rc=$?
done
