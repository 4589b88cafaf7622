# round-2 measurement: GPU tests, smoke, bench lines (all configs + reference arm),
# launch list of the default bench, ncu --set full of the dominant kernels
V=${V:-r2d}
O=gpurun_out/$V
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
for c in c1 c2 c4; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config c5 --scale 3 > $O/bench_c5s3.json 2> $O/bench_c5s3.err
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
timeout 900 python bench.py --impl reference --config c2 --steps 2 --warmup 1 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err
timeout 900 python bench.py --impl reference --config c4 --steps 2 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
python tools/launches.py $O/launches_c3.csv > $O/launches_c3.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_hash_probe_staged|k_bin_scatter_est|k_est_sample" -c 3 -o $O/full_c3 python tools/one_step.py c3 buffered 1 > $O/full_c3.log 2>&1
python tools/ncu_export.py $O/full_c3.ncu-rep c3 r02_ncu_full_c3 k_hash_probe_staged $O
python tools/ncu_sum.py $O/full_c3.ncu-rep > $O/sum_c3.txt 2>&1
timeout 900 $NCU -k regex:"k_grmi_probe_staged|k_bin_scatter_est|k_est_sample" -c 3 -o $O/full_c2 python tools/one_step.py c2 buffered 1 > $O/full_c2.log 2>&1
python tools/ncu_export.py $O/full_c2.ncu-rep c2 r02_ncu_full_c2 k_grmi_probe_staged $O
python tools/ncu_sum.py $O/full_c2.ncu-rep > $O/sum_c2.txt 2>&1
timeout 1200 $NCU -k regex:"k_lsj_sort|k_split_count|k_split_scatter|k_bin_scatter_est|k_est_sample|k_lsj_join" -c 20 -o $O/full_c4 python tools/one_step.py c4 x 1 > $O/full_c4.log 2>&1
python tools/ncu_export.py $O/full_c4.ncu-rep c4 r02_ncu_full_c4 k_lsj_sort $O
python tools/ncu_sum.py $O/full_c4.ncu-rep > $O/sum_c4.txt 2>&1
rm -f $O/full_c4.ncu-rep $O/full_c2.ncu-rep
du -sh $O
