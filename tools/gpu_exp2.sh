# experiment: LSJ coarse bin count, join occupancy variants
O=gpurun_out/exp2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
F='^c4|k_lsj_sort|k_bin_scatter|k_split|k_lsj_join|k_join_bounds|k_est_sample'
for nb in 2048 1024 512; do echo "== max bins $nb" >> $O/bins.txt; LJ_LSJ_MAX_BINS=$nb python tools/kprof.py c4 2>&1 | grep -E "$F" | cut -c1-90 >> $O/bins.txt; done
rm -rf gpurun_out/var
bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "-DLJ_JOIN_MINB=12 -DLJ_JOIN_WCAP=1024" "-DLJ_JOIN_MINB=10" "-DLJ_JOIN_NT=256 -DLJ_JOIN_T=1024 -DLJ_JOIN_MINB=5" "-DLJ_JOIN_T=256 -DLJ_JOIN_NT=64 -DLJ_JOIN_WCAP=1024 -DLJ_JOIN_MINB=16" "-DLJ_JOIN_T=1024 -DLJ_JOIN_NT=128 -DLJ_JOIN_WCAP=1920"
grep -E "^==|k_lsj_join|k_join_bounds|^c4" gpurun_out/var/out.txt | cut -c1-100 > $O/variants.txt
cp gpurun_out/var/err.txt $O/variants.err 2>/dev/null
