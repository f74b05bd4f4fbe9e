timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo exit=$? >> gpurun_out/bench_c3.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
