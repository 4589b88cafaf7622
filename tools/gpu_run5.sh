NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"k_bin_scatter_est" -c 1 -o gpurun_out/ncu_c2b python tools/one_step.py c2 buffered 1 > gpurun_out/ncu_c2b.log 2>&1
timeout 900 $NCU -k regex:"k_bin_hist_tma|k_bin_scatter_tma" -c 2 -o gpurun_out/ncu_c4b python tools/one_step.py c4 x 1 > gpurun_out/ncu_c4b.log 2>&1
