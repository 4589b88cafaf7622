# quick validation: GPU tests, per-kernel times of C3 / C2 / C4 (+ optional -D variants of lj_lsj.cu in $VARS)
O=gpurun_out/quick
mkdir -p $O
rm -rf gpurun_out/var
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in c3 c2 c4; do python tools/kprof.py $c > $O/kprof_$c.txt 2>&1; done
if [ -n "${VARS:-}" ]; then bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "$VARS"; cp gpurun_out/var/out.txt $O/variants.txt; fi
