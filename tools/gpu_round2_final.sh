# round-2 final evidence on one B200: smoke, every -m gpu test, the bench lines (default as the driver runs it,
# reference arm, C3); then -- each only after its plain command exited 0 -- the ncu captures: K1 / K2 of the constant
# path with the deferred x update (K1, K2 with x, K1, K2 without x), the symmetric C4 load, and the launch list of the
# bench command itself; the fused true-residual + EXP_true pass
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --timeout 1200 -rA > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo exit=$? >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo exit=$? >> gpurun_out/bench_reference.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo exit=$? >> gpurun_out/bench_c3.log
timeout 300 python tools/ncu_step.py --config c4 --skip-run --iters 4 > gpurun_out/plain_c4.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_const_tma --launch-skip 3 --launch-count 4 -o gpurun_out/p_const_xdefer python tools/ncu_step.py --config c4 --skip-run --iters 4 > gpurun_out/ncu_pc.log 2>&1
timeout 300 python tools/exp_timing.py 8 run > gpurun_out/exp_timing_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rhs_c4_sym -c 1 -o gpurun_out/rhs_c4_sym python tools/exp_timing.py 8 run > gpurun_out/ncu_rhs_sym.log 2>&1
# the finest level's true-residual pass in its EXP_true form (ECMG_OPT_RICH_FUSED): one ecmg_run inside the profiler range
timeout 300 python tools/ncu_step.py --config c4 --iters 1 --host-loop > gpurun_out/plain_c4_run.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_jcg_const_tma<\(int\)4, \(int\)4, \(int\)3>' --launch-count 1 -o gpurun_out/true_rich python tools/ncu_step.py --config c4 --iters 1 --host-loop > gpurun_out/ncu_tr.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-arrays > gpurun_out/bench_for_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-arrays > gpurun_out/ncu_lbench.log 2>&1
