timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/b20_c4.json 2> gpurun_out/b20_c4.err
