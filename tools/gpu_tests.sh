timeout 240 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staged or buffered or config2 or registry" > gpurun_out/pytest_gpu_a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_a.log
timeout 200 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/b_c2w.json 2> gpurun_out/b_c2w.err
