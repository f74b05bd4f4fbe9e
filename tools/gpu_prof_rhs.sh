timeout 300 python tools/ncu_step.py --config c4 --iters 0 > gpurun_out/plain_c4.log 2>&1 || exit 1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_rhs_c4 --launch-skip 7 --launch-count 1 -o gpurun_out/ps_rhs python tools/ncu_step.py --config c4 --iters 0 > gpurun_out/ncu_rhs.log 2>&1
