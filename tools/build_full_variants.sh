# full libecmg builds that differ in preprocessor flags: tools/build_full_variants.sh NAME "-DFLAGS" ...
#   -> vtmp/variants/libfull_NAME.so
set -e
cd "$(dirname "$0")/.."
FL="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared"
mkdir -p vtmp/variants
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  nvcc $FL $flags -o vtmp/variants/libfull_$name.so paper_1506_02983_b200/csrc/*.cu &
done; wait
