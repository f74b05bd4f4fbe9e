# quick GPU check: parity subset + bench lines
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -k "setup_ahead or ecmg_run or fullsize or slab or paper or exp or rhs" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
timeout 600 python tools/tune_setup.py > gpurun_out/tune_setup.log 2>&1
