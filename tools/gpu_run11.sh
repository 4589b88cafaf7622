LJ_STAGE_TRACE=gpurun_out/stage_trace.bin timeout 600 python tools/one_step.py c2 buffered 2 > gpurun_out/trace_c2.log 2>&1
python tools/stage_trace.py gpurun_out/stage_trace.bin >> gpurun_out/trace_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lsj_launches2.csv python tools/one_step.py c4 x 1 > gpurun_out/lsj_ncu2.log 2>&1
