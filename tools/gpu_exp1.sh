# experiment: compacted forward scan in the staged C3 probe
O=gpurun_out/exp1
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "hash or spline or c3 or registry or fullsize" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
python tools/kprof.py c3 > $O/kprof_c3_default.txt 2>&1
rm -rf gpurun_out/var
bash tools/gpu_variants.sh lj_hash_staged.cu "python tools/kprof.py c3" "-DLJ_HS_ROUNDS=1" "-DLJ_HS_ROUNDS=2 -DLJ_HS_NT=512 -DLJ_HS_U=3" "-DLJ_HS_ROUNDS=2 -DLJ_HS_NT=256 -DLJ_HS_CTAS=3" "-DLJ_HS_ROUNDS=2 -DLJ_HS_D=3 -DLJ_HS_U=2 -DLJ_HS_NT=512"
grep -E "^==|k_hash_probe_staged|of kernels" gpurun_out/var/out.txt > $O/variants.txt
cp gpurun_out/var/err.txt $O/variants.err 2>/dev/null
