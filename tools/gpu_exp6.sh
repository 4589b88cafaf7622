O=gpurun_out/exp6
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python tools/kprof.py c4 > $O/kprof_c4.txt 2>&1
python tools/kprof.py c2 > $O/kprof_c2.txt 2>&1
python tools/kprof.py c3 > $O/kprof_c3.txt 2>&1
python tools/kprof.py c5 > $O/kprof_c5.txt 2>&1
python tools/lsj_over.py > $O/lsj_over.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_hash_probe_staged|k_bin_scatter_est" -c 2 -o $O/c3 python tools/one_step.py c3 buffered 1 > $O/c3.log 2>&1
timeout 1200 $NCU -k regex:"k_grmi_probe_staged" -c 1 -o $O/c2 python tools/one_step.py c2 buffered 1 > $O/c2.log 2>&1
