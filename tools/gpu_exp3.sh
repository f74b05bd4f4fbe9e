timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing.log 2>&1; echo exit=$? >> gpurun_out/exp_timing.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "exp or rhs or setup_ahead or ecmg_run or smoke" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python tools/tune_setup.py 0 > gpurun_out/tune_setup.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_fused -c 1 -o gpurun_out/exp_fused python tools/exp_timing.py 8 exp1 > gpurun_out/ncu_exp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rhs_c4 -c 1 -o gpurun_out/rhs_c4 python tools/exp_timing.py 8 rhs > gpurun_out/ncu_rhs.log 2>&1
