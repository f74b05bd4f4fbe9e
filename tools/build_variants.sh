# build libecmg variants that differ only in kernels_jcg_elem.cu macros:
#   tools/build_variants.sh NAME "-DFLAGS" [NAME "-DFLAGS" ...]  ->  gpurun_out/variants/lib_NAME.so
set -e
cd "$(dirname "$0")/.."
OUT=build/variants; mkdir -p $OUT/common $OUT/elem
FL="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC"
for f in paper_1506_02983_b200/csrc/*.cu; do
  b=$(basename $f .cu); [ "$b" = kernels_jcg_elem ] && continue
  [ $OUT/common/$b.o -nt $f ] || nvcc $FL -c $f -o $OUT/common/$b.o &
done; wait
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  nvcc $FL $flags -c paper_1506_02983_b200/csrc/kernels_jcg_elem.cu -o $OUT/elem/$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib_$name.so $OUT/common/*.o $OUT/elem/$name.o
done
