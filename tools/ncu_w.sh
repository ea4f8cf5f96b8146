W=${W:-C4}
python tools/one_search.py $W > gpurun_out/plain_$W.log 2>&1
cap() { # kernel wave out
if [ -n "$2" ]; then python tools/one_search.py $W --target $1 --wave $2 > gpurun_out/t_$3.txt 2>&1
else python tools/one_search.py $W --target $1 > gpurun_out/t_$3.txt 2>&1; fi
SKIP=$(grep -o "skip [0-9]*" gpurun_out/t_$3.txt | awk '{print $2}')
ncu --set full --clock-control none --import-source on -k regex:"^$1\$|$1\(" -s $SKIP -c 1 -o gpurun_out/$3 python tools/one_search.py $W > gpurun_out/ncu_$3.log 2>&1; echo $3 rc=$?
}
cap k_filter "" cur_c4_filter
