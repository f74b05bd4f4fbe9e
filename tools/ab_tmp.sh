mkdir -p gpurun_out
: > gpurun_out/ab_tree.log
for r in 1 2; do for v in base tree tree_minb3; do timeout 300 python tools/tune_elem.py --one build/variants/libfull_$v.so c3 >> gpurun_out/ab_tree.log 2>&1; timeout 300 python tools/tune_elem.py --one build/variants/libfull_$v.so c5 >> gpurun_out/ab_tree.log 2>&1; done; done
