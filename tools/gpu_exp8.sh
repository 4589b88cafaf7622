O=gpurun_out/exp8
mkdir -p $O
rm -rf gpurun_out/var
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
python tools/kprof.py c5 > $O/kprof_c5.txt 2>&1
bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "-DLJ_SORT_CTAS=4" "-DLJ_SORT_CTAS=4 -DLJ_SORT_E=10"
cp gpurun_out/var/out.txt $O/variants.txt; cp gpurun_out/var/err.txt $O/variants.err
rm -rf gpurun_out/var
bash tools/gpu_variants.sh lj_hash_staged.cu "python tools/kprof.py c3" "-DLJ_HS_SPREAD=4" "-DLJ_HS_SPREAD=3"
cp gpurun_out/var/out.txt $O/variants_hs.txt; cp gpurun_out/var/err.txt $O/variants_hs.err
