timeout 400 python tools/tune_elem.py --zc paper_1506_02983_b200/libecmg.so c4 0 171 0 171 0 > gpurun_out/tune_elem.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "tma or graph or ecmg_run or fullsize" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
