# quick GPU check: slab / graph / parity subset
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -k "slab or graph_loop or hybrid or nccl or ecmg_run" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
