O=gpurun_out/psort
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_lsj_sort|k_bin_scatter_est" -c 6 -o $O/c4 python tools/one_step.py c4 x 1 > $O/c4.log 2>&1
python tools/ncu_sum.py $O/c4.ncu-rep > $O/c4_sum.txt 2>&1
