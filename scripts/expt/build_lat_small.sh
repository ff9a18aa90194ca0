# Variants of sb_reduce.cu for the small/mid-n latency A/B (scripts/expt/run_lat_small.py):
#   old  = the committed kernel (git HEAD), new = working tree,
#   tma0 = working tree with the TMA ring at every size.
set -e
cd "$(dirname "$0")/../.."
python -m paper_2009_10917_b200.build >/dev/null
OUT=scripts/expt/_lat2; mkdir -p $OUT
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC --expt-relaxed-constexpr -I$(python -c 'from paper_2009_10917_b200.build import nccl_include as f; print(f())')"
OBJS=$(ls paper_2009_10917_b200/build/*.o | grep -v sb_reduce)
SRC=paper_2009_10917_b200/csrc
git show HEAD:$SRC/sb_reduce.cu > $OUT/old_reduce.cu
$NV $FL -I$SRC -c $OUT/old_reduce.cu -o $OUT/old.o &
$NV $FL -c $SRC/sb_reduce.cu -o $OUT/new.o &
$NV $FL -DSB_TMA_MIN_FUSED=0 -DSB_TMA_MIN_DOT=0 -DSB_TMA_MIN_NORM=0 -c $SRC/sb_reduce.cu -o $OUT/tma0.o &
wait
for v in old new tma0; do
  [ -f $OUT/$v.o ] && $NV -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$v.so $OUT/$v.o $OBJS -cudart static -ldl
done
ls $OUT/*.so
