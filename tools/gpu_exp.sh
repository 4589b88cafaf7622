# round-2 session A: generator parity + C3 grouping experiment
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_inputs.py -x -q > gpurun_out/pytest_inputs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_inputs.log
for kb in "" 1; do for nb in 2048 1024 512 256; do
  env ${kb:+LJ_HASH_KEYBIN=1} LJ_HASH_BINS=$nb timeout 300 python tools/exp_c3_bins.py >> gpurun_out/exp_c3_bins.jsonl 2>> gpurun_out/exp_c3_bins.err
done; done
