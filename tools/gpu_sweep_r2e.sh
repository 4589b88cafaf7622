# build-constant sweep at HEAD: C3 probe and C4 LSJ kernels (one line per variant in gpurun_out/var/out.txt)
rm -rf gpurun_out/var
bash tools/gpu_variants.sh lj_hash_staged.cu "python tools/kprof.py c3 buffered 2" \
  "-DLJ_HS_SPREAD=2" "-DLJ_HS_SPREAD=3" "-DLJ_HS_PIECE=16384" "-DLJ_HS_PIECE=65536" \
  "-DLJ_HS_NT=256 -DLJ_HS_CTAS=3" "-DLJ_HS_NT=512 -DLJ_HS_CTAS=1 -DLJ_HS_U=4" "-DLJ_HS_U=2 -DLJ_HS_D=3 -DLJ_HS_CTAS=3" \
  "-DLJ_HS_U=3" "-DLJ_HS_NC=2048" "-DLJ_HS_NT=320 -DLJ_HS_CTAS=2 -DLJ_HS_U=5"
bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4 x 2" \
  "-DLJ_SORT_CTAS=5" "-DLJ_SORT_NT=128 -DLJ_SORT_E=8 -DLJ_SORT_CTAS=10" "-DLJ_SORT_NT=128 -DLJ_SORT_E=16 -DLJ_SORT_CTAS=5" \
  "-DLJ_SORT_NT=512 -DLJ_SORT_E=4 -DLJ_SORT_CTAS=3" "-DLJ_SORT_U=2" "-DLJ_SUB_DIV=3 -DLJ_SORT_E=12 -DLJ_SORT_CTAS=3" \
  "-DLJ_JOIN_T=1024" "-DLJ_JOIN_NT=256" "-DLJ_SPLIT_U=8" "-DLJ_SPLIT_U=2"
grep -E "^==|ms of kernels|k_hash_probe_staged|k_lsj_sort<|k_split_scatter|k_split_count|k_lsj_join|words" gpurun_out/var/out.txt > gpurun_out/var/summary.txt
