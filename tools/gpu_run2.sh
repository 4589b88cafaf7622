timeout 900 python tools/exp_c3.py > gpurun_out/exp_c3.log 2>&1
timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lsj_launches.csv python tools/lsj_phases.py c4 > gpurun_out/lsj_ncu.log 2>&1
