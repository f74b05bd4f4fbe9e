# A/B of library variants (vtmp/variants/libfull_NAME.so) on the JCG iteration: tools/gpu_ab.sh "cfg1 cfg2" NAME1 NAME2 ...
# two interleaved rounds per config; one JSON line per (variant, config) in gpurun_out/ab.log
mkdir -p gpurun_out
cfgs=$1; shift
for round in 1 2; do
  for c in $cfgs; do
    for v in "$@"; do
      timeout 300 python tools/tune_elem.py --one vtmp/variants/libfull_$v.so $c >> gpurun_out/ab.log 2>&1
    done
  done
done
