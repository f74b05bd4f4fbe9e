timeout 300 python tools/exp_timing.py 8 run > gpurun_out/exp_timing.log 2>&1; echo exit=$? >> gpurun_out/exp_timing.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_fused --launch-skip 5 -c 1 -o gpurun_out/exp_fused_fb python tools/exp_timing.py 8 run > gpurun_out/ncu_exp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_interp --launch-skip 5 -c 1 -o gpurun_out/exp_interp_fb python tools/exp_timing.py 8 run > gpurun_out/ncu_exp2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_seeds --launch-skip 5 -c 1 -o gpurun_out/exp_seeds_fb python tools/exp_timing.py 8 run > gpurun_out/ncu_exp3.log 2>&1
