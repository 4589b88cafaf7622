O=gpurun_out/exp4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "lsj or multi or dist or cabi" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
LJ_LSJ_ONE_STREAM=1 timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4_one.json 2> $O/bench_c4_one.err
