# Build libsb200 variants with different lattice ring shapes for run_lattice.py
# (run here; the .so files travel to the box with the snapshot).
set -e
cd "$(dirname "$0")/../.."
python -m paper_2009_10917_b200.build >/dev/null
OUT=scripts/expt/_lat; mkdir -p $OUT
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC --expt-relaxed-constexpr -I$(python -c 'from paper_2009_10917_b200.build import nccl_include as f; print(f())')"
OBJS=$(ls paper_2009_10917_b200/build/*.o | grep -v sb_reduce)
while read name sn sd sf rn rd rf bpc rfb; do
  [ -z "$name" ] && continue
  $NV $FL -DSB_SPS_NORM=$sn -DSB_SPS_DOT=$sd -DSB_SPS_FUSED=$sf -DSB_RING_NORM=$rn -DSB_RING_DOT=$rd \
      -DSB_RING_FUSED=$rf -DSB_BPC=${bpc:-1} -DSB_RING_FUSED_BPC4=${rfb:-131072} -c paper_2009_10917_b200/csrc/sb_reduce.cu -o $OUT/$name.o &
done < scripts/expt/lattice_variants.txt
wait
while read name rest; do
  [ -z "$name" ] && continue
  $NV -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $OUT/$name.o $OBJS -cudart static -ldl
done < scripts/expt/lattice_variants.txt
ls $OUT/*.so
