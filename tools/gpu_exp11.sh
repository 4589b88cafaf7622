O=gpurun_out/exp11
mkdir -p $O
rm -rf gpurun_out/var
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "lsj" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "-DLJ_JOIN_T=512 -DLJ_JOIN_WCAP=1920" "-DLJ_JOIN_T=512 -DLJ_JOIN_WCAP=1920 -DLJ_JOIN_NT=128" "-DLJ_JOIN_T=2048 -DLJ_JOIN_WCAP=3840 -DLJ_JOIN_NT=512"
cp gpurun_out/var/out.txt $O/variants.txt; cp gpurun_out/var/err.txt $O/variants.err
