timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s --timeout 900 > gpurun_out/gpu_full.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_full.log
