# round measurement: benches (all configs + reference arm), launch list, ncu --set full of the dominant kernels
V=${V:-v12}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$V.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$V.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$V.log
for c in c2 c1 c3 c4; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$V.json 2> gpurun_out/bench_${c}_$V.err; done
timeout 900 python bench.py --config c5 --scale 3 --no-cpu-baseline > gpurun_out/bench_c5s3_$V.json 2> gpurun_out/bench_c5s3_$V.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$V.json 2> gpurun_out/bench_ref_$V.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_$V.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$V.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"k_grmi_probe_staged|k_bin_scatter_est|k_est_sample" -c 3 -o gpurun_out/full_c2_$V python tools/one_step.py c2 buffered 1 > gpurun_out/full_c2_$V.log 2>&1
timeout 900 $NCU -k regex:"k_grmi_probe" -c 1 -o gpurun_out/full_c1_$V python tools/one_step.py c1 direct 1 > gpurun_out/full_c1_$V.log 2>&1
timeout 1200 $NCU -k regex:"k_hash_probe_chunks|k_bin_scatter_est|k_est_sample" -c 3 -o gpurun_out/full_c3_$V python tools/one_step.py c3 buffered 1 > gpurun_out/full_c3_$V.log 2>&1
timeout 1200 $NCU -k regex:"k_lsj_sort|k_split_count|k_split_scatter|k_bin_scatter_est|k_est_sample|k_lsj_join" -c 12 -o gpurun_out/full_c4_$V python tools/one_step.py c4 x 1 > gpurun_out/full_c4_$V.log 2>&1
# summaries on the box (the .ncu-rep files are too large to bring back)
mkdir -p gpurun_out/prof_$V
python tools/ncu_export.py gpurun_out/full_c2_$V.ncu-rep c2 r01_ncu_full_c2_$V k_grmi_probe_staged gpurun_out/prof_$V
python tools/ncu_export.py gpurun_out/full_c1_$V.ncu-rep c1 r01_ncu_full_c1_$V k_grmi_probe gpurun_out/prof_$V
python tools/ncu_export.py gpurun_out/full_c3_$V.ncu-rep c3 r01_ncu_full_c3_$V k_hash_probe_chunks gpurun_out/prof_$V
python tools/ncu_export.py gpurun_out/full_c4_$V.ncu-rep c4 r01_ncu_full_c4_$V k_lsj_sort gpurun_out/prof_$V
for c in c2 c3 c4; do python tools/ncu_sum.py gpurun_out/full_${c}_$V.ncu-rep > gpurun_out/prof_$V/sum_$c.txt 2>&1; done
python tools/ncu_src.py gpurun_out/full_c4_$V.ncu-rep k_lsj_join 30 > gpurun_out/prof_$V/src_c4_join.txt 2>&1
python tools/ncu_src.py gpurun_out/full_c4_$V.ncu-rep k_lsj_sort 30 > gpurun_out/prof_$V/src_c4_sort.txt 2>&1
python tools/ncu_src.py gpurun_out/full_c3_$V.ncu-rep k_hash_probe_chunks 30 > gpurun_out/prof_$V/src_c3_probe.txt 2>&1
rm -f gpurun_out/full_c3_$V.ncu-rep gpurun_out/full_c4_$V.ncu-rep gpurun_out/full_c1_$V.ncu-rep
du -sh gpurun_out
