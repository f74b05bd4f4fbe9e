timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.log 2>&1; echo bench_exit=$? >> gpurun_out/bench2.log
timeout 300 python tools/ncu_step.py > gpurun_out/ncu_step_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_step.py > gpurun_out/ncu_launches.log 2>&1; echo ncu1_exit=$? >> gpurun_out/ncu_launches.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_const -c 4 -o gpurun_out/prof_jcg python tools/ncu_step.py --skip-run --iters 2 > gpurun_out/ncu_full.log 2>&1; echo ncu2_exit=$? >> gpurun_out/ncu_full.log
tail -2 gpurun_out/gpu_tests.log
