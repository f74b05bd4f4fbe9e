mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_arrays.py tests/test_gpu_paper.py tests/test_gpu_slabs.py "tests/test_gpu_fullsize_golden.py::test_alg4_fullsize_vs_oracle[c3]" "tests/test_gpu_fullsize_golden.py::test_alg4_fullsize_vs_oracle[c5_256]" tests/test_gpu_fullsize.py -m gpu -q --timeout 900 -rA > gpurun_out/elem80_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/elem80_tests.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
