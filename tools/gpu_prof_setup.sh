timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/ncu_step.py > gpurun_out/ncu_step_plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_rhs|k_exp_finite|k_exp_true|k_gather|k_scatter" -c 40 -o gpurun_out/prof_setup python tools/ncu_step.py --iters 1 > gpurun_out/ncu_setup.log 2>&1; echo ncu_exit=$? >> gpurun_out/ncu_setup.log
tail -2 gpurun_out/gpu_tests.log
