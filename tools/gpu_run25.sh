for v in 1 2; do LJ_LIB=paper_2111_08824_b200/csrc/variants/liblj_sort$v.so timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases25_$v.log 2>&1; done
timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases25_4.log 2>&1
