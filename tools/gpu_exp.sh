# EXP_finite: parity tests, timings at 512^3 (default build and variants named on the command line), ncu of the
# fused kernel inside ecmg_run
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "exp and not golden" --timeout 600 > gpurun_out/exp_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/exp_tests.log
timeout 300 python tools/exp_timing.py 8 > gpurun_out/exp_timing.log 2>&1
for v in "$@"; do echo "== $v" >> gpurun_out/exp_timing.log; ECMG_LIB_PATH=$PWD/vtmp/variants/libfull_$v.so timeout 300 python tools/exp_timing.py 8 run >> gpurun_out/exp_timing.log 2>&1; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_fused --launch-skip 5 -c 1 -o gpurun_out/exp_fused_r2 python tools/exp_timing.py 8 run > gpurun_out/ncu_exp.log 2>&1
