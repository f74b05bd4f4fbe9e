timeout 300 python tools/exp_timing.py 8 rich > gpurun_out/exp_timing.log 2>&1; timeout 300 python tools/exp_timing.py 8 rich >> gpurun_out/exp_timing.log 2>&1; echo exit=$? >> gpurun_out/exp_timing.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "exp_true or ecmg_run or fullsize_exp or slab_run" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_true -c 1 -o gpurun_out/exp_true python tools/exp_timing.py 8 rich > gpurun_out/ncu_rich.log 2>&1
