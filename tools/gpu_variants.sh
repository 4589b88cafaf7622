# build -D variants of one source file and run a command with each:
#   bash tools/gpu_variants.sh lj_lsj.cu "python tools/kprof.py c4" "-DLJ_SORT_CTAS=5" "-DLJ_SORT_E=8 -DLJ_SORT_NT=384"
set -u
SRC=$1; CMD=$2; shift 2
O=gpurun_out/var
mkdir -p $O
C=paper_2111_08824_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -I include"
OBJS=$(ls $C/build/*.o | grep -v "$SRC")
for v in "$@"; do
  tag=$(echo "$SRC $v" | tr ' =.' '___')
  mkdir -p /tmp/var_$tag
  nvcc $ARCH $FL $v -c $C/$SRC -o /tmp/var_$tag/v.o >> $O/build.log 2>&1
  nvcc $ARCH -shared -o /tmp/var_$tag/lib.so $OBJS /tmp/var_$tag/v.o -cudart static >> $O/build.log 2>&1
  echo "== $SRC $v" >> $O/out.txt
  LJ_LIB=/tmp/var_$tag/lib.so timeout 600 $CMD >> $O/out.txt 2>> $O/err.txt
done
