NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"k_bin_scatter_est|k_grmi_probe_staged|k_est_sample" -c 3 -o gpurun_out/ncu_c2 python tools/one_step.py c2 buffered 2 > gpurun_out/ncu_c2.log 2>&1
timeout 900 $NCU -k regex:"k_bin_hist_tma|k_bin_scatter_tma|k_lsj_sort|k_lsj_join|k_split_count|k_split_scatter" -c 10 -o gpurun_out/ncu_c4 python tools/one_step.py c4 x 2 > gpurun_out/ncu_c4.log 2>&1
