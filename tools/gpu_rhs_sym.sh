# the permutation-symmetric C4 load: parity tests, its time alone, and the A/B of the C4 step
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "rhs" -rA -s > gpurun_out/rhs_sym_tests.log 2>&1; echo exit=$? >> gpurun_out/rhs_sym_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fullsize_golden.py -m gpu -q -k "rhs or c4 or C4" -rA >> gpurun_out/rhs_sym_tests.log 2>&1; echo exit=$? >> gpurun_out/rhs_sym_tests.log
timeout 300 python tools/exp_timing.py 8 rhs > gpurun_out/rhs_sym_timing.log 2>&1
timeout 600 python tools/tts_ab.py 15 RHS_SYM=248 RHS_SYM=0 > gpurun_out/ab_rhs_sym.log 2>&1
