timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases19.log 2>&1
LJ_PART_RECOMPUTE=1 timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases19r.log 2>&1
timeout 900 python tools/exp_c3.py > gpurun_out/exp_c3_19.log 2>&1
