# build variants of the staged C3 probe (-D constants) and time each with tools/exp_c3_bins.py
set -u
mkdir -p gpurun_out/hv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hv/build.log 2>&1
C=paper_2111_08824_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -I include"
OBJS=$(ls $C/build/*.o | grep -v lj_hash_staged)
for v in "$@"; do
  tag=$(echo "$v" | tr ' =' '_-')
  mkdir -p /tmp/hv_$tag
  nvcc $ARCH $FL $v -c $C/lj_hash_staged.cu -o /tmp/hv_$tag/hs.o >> gpurun_out/hv/build.log 2>&1
  nvcc $ARCH -shared -o /tmp/hv_$tag/lib.so $OBJS /tmp/hv_$tag/hs.o -cudart static >> gpurun_out/hv/build.log 2>&1
  echo "== $v" >> gpurun_out/hv/exp.jsonl
  LJ_LIB=/tmp/hv_$tag/lib.so timeout 300 python tools/exp_c3_bins.py >> gpurun_out/hv/exp.jsonl 2>> gpurun_out/hv/exp.err
done
