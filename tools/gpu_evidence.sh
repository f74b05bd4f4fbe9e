# round evidence: GPU tests, bench lines (default as the driver runs it, reference arm, C3), ncu K1/K2
# captures + launch lists (tools/gpu_profiles.sh), setup / EXP kernel captures at 512^3, and the ncu
# launch list of the bench command itself
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo exit=$? >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo exit=$? >> gpurun_out/bench_reference.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo exit=$? >> gpurun_out/bench_c3.log
bash tools/gpu_profiles.sh > gpurun_out/profiles_run.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_fused --launch-skip 5 -c 1 -o gpurun_out/exp_fused_fb python tools/exp_timing.py 8 run > gpurun_out/ncu_exp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rhs_c4 -c 1 -o gpurun_out/rhs_c4 python tools/exp_timing.py 8 rhs > gpurun_out/ncu_rhs.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_true -c 1 -o gpurun_out/exp_true python tools/exp_timing.py 8 rich > gpurun_out/ncu_rich.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_lbench.log 2>&1
# the fusion ablation: per-launch time and DRAM bytes of 3 fused and 3 unfused (textbook) 512^3 iterations
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_fused3.csv python tools/ncu_step.py --config c4 --skip-run --iters 3 > gpurun_out/ncu_lf.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_unfused3.csv python tools/ncu_step.py --config c4 --skip-run --iters 3 --unfused > gpurun_out/ncu_lu.log 2>&1
