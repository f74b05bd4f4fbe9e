# quick GPU check: parity subset + one bench line
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -k "ecmg_run or persistent or cta or slab or paper or fullsize or setup_ahead" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
