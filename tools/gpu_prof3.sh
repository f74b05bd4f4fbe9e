timeout 300 python tools/ncu_step.py > gpurun_out/ncu_step_plain.log 2>&1 || exit 1
N="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 600 $N -k regex:k_rhs_vol --launch-skip 7 --launch-count 1 -o gpurun_out/p_rhs2 python tools/ncu_step.py --iters 2 > gpurun_out/ncu_p3.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1
