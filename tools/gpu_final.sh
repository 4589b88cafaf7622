V=v15
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$V.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$V.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$V.log
timeout 600 python bench.py > gpurun_out/bench_default_$V.json 2> gpurun_out/bench_default_$V.err
for c in c1 c3 c4; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$V.json 2> gpurun_out/bench_${c}_$V.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$V.json 2> gpurun_out/bench_ref_$V.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_$V.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$V.log 2>&1
mkdir -p gpurun_out/prof_$V
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lsj_sort|k_split_count|k_split_scatter|k_lsj_join" -c 8 -o gpurun_out/full_c4_$V python tools/one_step.py c4 x 1 > gpurun_out/full_c4_$V.log 2>&1
python tools/ncu_export.py gpurun_out/full_c4_$V.ncu-rep c4 r01_ncu_full_c4_$V k_lsj_sort gpurun_out/prof_$V
python tools/ncu_sum.py gpurun_out/full_c4_$V.ncu-rep > gpurun_out/prof_$V/sum_c4.txt 2>&1
rm -f gpurun_out/full_c4_$V.ncu-rep
