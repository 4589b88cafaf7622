# run the small grouped-probe parity test against -D variants of lj_hash_staged.cu (bisecting a variant-only failure)
C=paper_2111_08824_b200/csrc
mkdir -p /tmp/vs gpurun_out/san
OBJS=$(ls $C/build/*.o | grep -v lj_hash_staged.cu)
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -I include $v -c $C/lj_hash_staged.cu -o /tmp/vs/v.o > gpurun_out/san/build.log 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/vs/lib.so $OBJS /tmp/vs/v.o -cudart static >> gpurun_out/san/build.log 2>&1
  echo "== $v"
  LJ_LIB=/tmp/vs/lib.so timeout 300 python -m pytest tests -m gpu -x -q -k "spline_hash_grouped" 2>&1 | tail -1
done
