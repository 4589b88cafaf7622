mkdir -p gpurun_out/timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/timing/build.log 2>&1
( time python bench.py > gpurun_out/timing/bench.json 2> gpurun_out/timing/bench.err ) 2> gpurun_out/timing/bench.time
( time python bench.py --impl reference > gpurun_out/timing/ref.json 2> gpurun_out/timing/ref.err ) 2> gpurun_out/timing/ref.time
