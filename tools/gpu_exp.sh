# C3 grouping experiment: direct claims scatter vs permuting claims scatter
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for d in 1 ""; do for kb in "" 1; do for nb in 2048 1024 512 256; do
  env ${d:+LJ_HASH_DIRECT=1} ${kb:+LJ_HASH_KEYBIN=1} LJ_HASH_BINS=$nb timeout 300 python tools/exp_c3_bins.py >> gpurun_out/exp_c3_bins2.jsonl 2>> gpurun_out/exp_c3_bins2.err
done; done; done
