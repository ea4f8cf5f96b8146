python tools/one_search.py C5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_plan -s 3 -c 1 -o gpurun_out/prof_c5_plan python tools/one_search.py C5 > gpurun_out/ncu_plan.log 2>&1; echo rc=$?
