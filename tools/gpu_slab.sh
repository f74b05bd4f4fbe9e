timeout 1200 python -m pytest tests/test_gpu_slabs.py -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -k "ecmg_run or cta or persistent or setup_ahead" >> gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
