timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.log 2>&1; echo bench_exit=$? >> gpurun_out/bench3.log
timeout 300 python tools/ncu_step.py > gpurun_out/ncu_step_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_step.py > gpurun_out/ncu_launches.log 2>&1; echo ncu1_exit=$? >> gpurun_out/ncu_launches.log
tail -2 gpurun_out/gpu_tests.log
