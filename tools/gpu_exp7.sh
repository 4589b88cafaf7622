O=gpurun_out/exp7
mkdir -p $O
rm -rf gpurun_out/var
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
python tools/kprof.py c3 > $O/kprof_c3.txt 2>&1
python tools/kprof.py c2 > $O/kprof_c2.txt 2>&1
bash tools/gpu_variants.sh lj_lsj.cu "python tools/one_step.py c4 x 1" "-DLJ_SORT_DIAG"
grep "^over" gpurun_out/var/out.txt | sort | uniq -c | sort -k3,3n -k4,4n | head -4000 > $O/over.txt
