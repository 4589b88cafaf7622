O=gpurun_out/exp9
mkdir -p $O
rm -rf gpurun_out/var
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "-DLJ_SPLIT_MINB=2" "-DLJ_SPLIT_MINB=2 -DLJ_SPLIT_U=2" "-DLJ_SPLIT_U=2"
cp gpurun_out/var/out.txt $O/variants.txt; cp gpurun_out/var/err.txt $O/variants.err
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_lsj_join|k_split_scatter" -c 3 -o $O/c4 python tools/one_step.py c4 x 1 > $O/c4.log 2>&1
python tools/ncu_sum.py $O/c4.ncu-rep > $O/c4_sum.txt 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
