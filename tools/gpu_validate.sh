# full validation on one B200: smoke, every -m gpu test, the default bench line and the reference arm
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --timeout 1200 -rA > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo exit=$? >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_reference.log 2>&1; echo exit=$? >> gpurun_out/bench_reference.log
