timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/b21_c2.json 2> gpurun_out/b20_c4.err
LJ_NO_STAGE_IMAGE=1 timeout 900 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/b21_c2_noimg.json 2> gpurun_out/b21_c2_noimg.err
