# round-2 profile evidence: K1 / K2 full captures (C4 constant, C3 element) + per-launch lists (tools/gpu_profiles.sh),
# the EXP_finite / EXP_true / RHS kernels at 512^3, and the launch list of the bench command itself
mkdir -p gpurun_out
bash tools/gpu_profiles.sh > gpurun_out/profiles_run.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_fused --launch-skip 5 -c 1 -o gpurun_out/exp_fused_r2 python tools/exp_timing.py 8 run > gpurun_out/ncu_exp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_true -c 1 -o gpurun_out/exp_true_r2 python tools/exp_timing.py 8 rich > gpurun_out/ncu_rich.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rhs_c4 -c 1 -o gpurun_out/rhs_c4_r2 python tools/exp_timing.py 8 rhs > gpurun_out/ncu_rhs.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-arrays > gpurun_out/bench_for_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-arrays > gpurun_out/ncu_lbench.log 2>&1
