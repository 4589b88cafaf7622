timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/b4_c2.json 2> gpurun_out/b4_c2.err
LJ_K4_MODEL_BINS=1 timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/b4_c2_model.json 2> gpurun_out/b4_c2_model.err
timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases4.log 2>&1
LJ_LSJ_MODEL_BINS=1 timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases4_model.log 2>&1
