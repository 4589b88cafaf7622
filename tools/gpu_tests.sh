timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/exp_c3.py > gpurun_out/exp_c3_p.log 2>&1
LJ_PART_NO_PIPE=1 timeout 900 python tools/exp_c3.py > gpurun_out/exp_c3_np.log 2>&1
