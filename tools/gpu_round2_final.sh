# round-2 re-validation on one B200 at HEAD: smoke, every -m gpu test, the default bench line, then (after those
# exited 0 without ncu) the K1/K2 captures with the deferred x update (4 launches: K1, K2 with x, K1, K2 without x)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --timeout 1200 -rA > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo exit=$? >> gpurun_out/bench_default.log
timeout 300 python tools/ncu_step.py --config c4 --skip-run --iters 4 > gpurun_out/plain_c4.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_const_tma --launch-skip 3 --launch-count 4 -o gpurun_out/p_const_xdefer python tools/ncu_step.py --config c4 --skip-run --iters 4 > gpurun_out/ncu_pc.log 2>&1
