timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases30.log 2>&1
for v in x2c4 x2c3 verify; do LJ_LIB=paper_2111_08824_b200/csrc/variants/liblj_$v.so timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases30_$v.log 2>&1; done
for v in x2c4 x2c3; do LJ_LIB=paper_2111_08824_b200/csrc/variants/liblj_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "lsj" > gpurun_out/pytest_lsj_$v.log 2>&1; done
