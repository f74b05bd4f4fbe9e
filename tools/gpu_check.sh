# quick GPU check: slab / parity subset
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -k "slab or hybrid or nccl or ecmg_run or setup_ahead" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
