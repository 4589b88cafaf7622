mkdir -p gpurun_out/c3dir
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c3dir/build.log 2>&1
python tools/exp_c3_bins.py > gpurun_out/c3dir/default.json 2> gpurun_out/c3dir/default.err
LJ_HASH_DIRECT=1 python tools/exp_c3_bins.py > gpurun_out/c3dir/direct.json 2> gpurun_out/c3dir/direct.err
LJ_HASH_BINS=256 python tools/exp_c3_bins.py > gpurun_out/c3dir/b256.json 2> gpurun_out/c3dir/b256.err
LJ_HASH_BINS=1024 python tools/exp_c3_bins.py > gpurun_out/c3dir/b1024.json 2> gpurun_out/c3dir/b1024.err
