timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -x -k "persistent or ecmg_run or tma or graph or cta or setup_ahead or slab or pdl" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/tune_setup.py 0 > gpurun_out/tune_setup.log 2>&1
