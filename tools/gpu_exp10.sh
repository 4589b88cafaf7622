O=gpurun_out/exp10
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
python tools/kprof.py c5 > $O/kprof_c5.txt 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
