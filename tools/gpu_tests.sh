timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c5 --scale 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
LJ_SHUFFLE=nccl timeout 900 python bench.py --config c5 --scale 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c5n.json 2> gpurun_out/b_c5n.err
