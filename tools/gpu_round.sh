# full GPU round: tests, smoke, bench, launch list, and full ncu of the setup / EXP kernels (512^3)
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_exit=$? >> gpurun_out/bench.log
timeout 300 python tools/ncu_step.py > gpurun_out/ncu_step_plain.log 2>&1 || exit 0
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_step.py > gpurun_out/ncu_launches.log 2>&1
N="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 600 $N -k regex:k_rhs_vol --launch-skip 7 --launch-count 1 -o gpurun_out/p_rhs python tools/ncu_step.py --iters 2 > gpurun_out/ncu_p.log 2>&1
timeout 600 $N -k regex:k_exp_true --launch-count 1 -o gpurun_out/p_exptrue python tools/ncu_step.py --iters 2 >> gpurun_out/ncu_p.log 2>&1
timeout 600 $N -k regex:k_exp_interp --launch-skip 5 --launch-count 1 -o gpurun_out/p_expint python tools/ncu_step.py --iters 2 >> gpurun_out/ncu_p.log 2>&1
