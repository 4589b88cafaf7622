timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/b23_c2.json 2> gpurun_out/b23_c2.err
timeout 300 python tools/lsj_phases.py c4 > gpurun_out/lsj_phases23.log 2>&1
timeout 900 python tools/exp_c3.py > gpurun_out/exp_c3_23.log 2>&1
