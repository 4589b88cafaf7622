NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_hash_probe|k_est_sample|k_bin_scatter_est" -c 4 -o gpurun_out/ncu_c3g python tools/one_step.py c3 buffered 1 > gpurun_out/ncu_c3g.log 2>&1
