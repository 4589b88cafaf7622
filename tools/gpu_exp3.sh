# record-source LSJ: tests + C5 bench line + C4 kernel times (regression check)
O=gpurun_out/exp3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "lsj or record or dist or c5 or part" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --config c5 --scale 3 --no-cpu-baseline > $O/bench_c5s3.json 2> $O/bench_c5s3.err
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
python tools/kprof.py c2 > $O/kprof_c2.txt 2>&1
