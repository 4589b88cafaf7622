LJ_LIB=paper_2111_08824_b200/csrc/variants/liblj_na.so timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases26_na.log 2>&1
timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases26.log 2>&1
