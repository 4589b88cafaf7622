# quick validation: GPU tests, per-kernel times of C4, a C4 bench line (+ optional -D variants of lj_lsj.cu in $VARS)
O=gpurun_out/quick
mkdir -p $O
rm -rf gpurun_out/var
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
if [ -n "${VARS:-}" ]; then bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "$VARS"; cp gpurun_out/var/out.txt $O/variants.txt; fi
