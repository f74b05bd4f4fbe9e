timeout 300 python tools/ncu_step.py > gpurun_out/ncu_step_plain.log 2>&1 || exit 1
N="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 600 $N -k regex:k_rhs_vol --launch-skip 7 --launch-count 1 -o gpurun_out/p_rhs python tools/ncu_step.py --iters 2 > gpurun_out/ncu_p.log 2>&1
timeout 600 $N -k regex:k_exp_true --launch-count 1 -o gpurun_out/p_exptrue python tools/ncu_step.py --iters 2 >> gpurun_out/ncu_p.log 2>&1
timeout 600 $N -k regex:k_exp_interp --launch-skip 5 --launch-count 1 -o gpurun_out/p_expint python tools/ncu_step.py --iters 2 >> gpurun_out/ncu_p.log 2>&1
timeout 600 $N -k regex:"k_jcg_const_tma" --launch-count 3 -o gpurun_out/p_jcg python tools/ncu_step.py --skip-run --iters 2 >> gpurun_out/ncu_p.log 2>&1
echo ncu_done >> gpurun_out/ncu_p.log
ls -la gpurun_out >> gpurun_out/ncu_p.log
