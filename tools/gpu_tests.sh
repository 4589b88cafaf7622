timeout 600 python tools/dbg_lsj.py tools/bad_5.pt > gpurun_out/dbg_lsj_fix.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
