timeout 300 python tools/exp_timing.py > gpurun_out/exp_timing.log 2>&1; echo exit=$? >> gpurun_out/exp_timing.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_fused -c 1 -o gpurun_out/exp_fused python tools/exp_timing.py 8 exp1 > gpurun_out/ncu_exp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rhs_c4 -c 1 -o gpurun_out/rhs_c4 python tools/exp_timing.py 8 rhs > gpurun_out/ncu_rhs.log 2>&1
