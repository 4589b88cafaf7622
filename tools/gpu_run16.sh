timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b16_c2.json 2> gpurun_out/b16_c2.err
