# C3-only re-measurement after a change to the staged probe: GPU tests, bench line, launch list, ncu --set full
V=${V:-r2h}
O=gpurun_out/$V
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
python tools/launches.py $O/launches_c3.csv > $O/launches_c3.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_hash_probe_staged|k_bin_scatter_est|k_est_sample" -c 3 -o $O/full_c3 python tools/one_step.py c3 buffered 1 > $O/full_c3.log 2>&1
python tools/ncu_export.py $O/full_c3.ncu-rep c3 r02_ncu_full_c3 k_hash_probe_staged $O
python tools/ncu_sum.py $O/full_c3.ncu-rep > $O/sum_c3.txt 2>&1
rm -f $O/full_c3.ncu-rep
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log; cat $O/bench_c3.json | cut -c1-400
