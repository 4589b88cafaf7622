mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "keybin or key_bounds or spline or config3 or lsj or hash" > gpurun_out/pytest_kb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_kb.log
for nb in 512 256 1024; do
  LJ_HASH_BINS=$nb timeout 300 python tools/exp_c3_bins.py >> gpurun_out/exp_c3_kb.jsonl 2>> gpurun_out/exp_c3_kb.err
done
