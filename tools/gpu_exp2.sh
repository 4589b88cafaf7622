# experiment round: GPU tests, C3 bucket/probe times (default and the slot-by-slot ablation), quick bench lines
O=gpurun_out/exp2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/exp_c3_bins.py > $O/c3_default.json 2> $O/c3_default.err
rm -f gpurun_out/hv/exp.jsonl
bash tools/gpu_hash_variants.sh "-DLJ_HS_ROUNDS=0"
cp gpurun_out/hv/exp.jsonl $O/c3_variants.jsonl
for c in c3 c2 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
