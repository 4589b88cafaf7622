timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for u in 1 2 4; do LJ_K1_ILP=$u timeout 200 python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/b_c1_$u.json 2> gpurun_out/b_c1_$u.err; done
