timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases24.log 2>&1
for u in 2 8; do for c in 4 6; do LJ_HASH_U=$u LJ_HASH_CTAS=$c timeout 900 python tools/exp_c3.py > gpurun_out/exp_c3_24_${u}_$c.log 2>&1; done; done
