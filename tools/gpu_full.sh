# full verification: GPU tests, smoke, bench (default C3) + reference arm
V=${V:-r2a}
mkdir -p gpurun_out/$V
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$V/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/$V/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$V/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$V/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$V/smoke.log
timeout 1200 python bench.py > gpurun_out/$V/bench_default.json 2> gpurun_out/$V/bench_default.err
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$V/bench_ref.json 2> gpurun_out/$V/bench_ref.err
nproc > gpurun_out/$V/nproc.txt; free -g >> gpurun_out/$V/nproc.txt
