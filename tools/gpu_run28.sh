NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"k_lsj_sort|k_split_scatter|k_split_count" -c 3 -o gpurun_out/ncu_sort python tools/one_step.py c4 x 1 > gpurun_out/ncu_sort.log 2>&1
