mkdir -p gpurun_out/lsj
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/lsj/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/lsj/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/lsj/pytest_gpu.log
timeout 600 python tools/lsj_diag.py > gpurun_out/lsj/lsj_diag.jsonl 2>&1
timeout 900 python bench.py --config c4 --no-e2e > gpurun_out/lsj/bench_c4.json 2> gpurun_out/lsj/bench_c4.err
