# cache-hint variants of the staged probe's slot-pair load
rm -rf gpurun_out/var
bash tools/gpu_variants.sh lj_hash_staged.cu "timeout 200 python tools/kprof.py c3 buffered 2" "-DLJ_HS_LDV=1" "-DLJ_HS_LDV=2" "-DLJ_HS_LDV=3" "-DLJ_HS_LDV=4" "-DLJ_HS_LDV=5"
grep -E "^==|k_hash_probe_staged|words" gpurun_out/var/out.txt | cut -c1-110; grep -i "error" gpurun_out/var/err.txt gpurun_out/var/build.log | head -3
