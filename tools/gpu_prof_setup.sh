# setup / EXP kernels of the C4 finest level (the last launch of each at 512^3): plain run, then one
# ncu --set full capture per kernel
timeout 300 python tools/ncu_step.py --config c4 --iters 0 > gpurun_out/plain_c4.log 2>&1 || exit 1
for spec in "k_rhs_c4 7" "k_rhs_shell 7" "k_exp_true 0" "k_exp_interp 5" "k_exp_seeds 5" "k_scatter 7"; do
  set -- $spec
  timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:"$1" --launch-skip $2 --launch-count 1 -o gpurun_out/ps_$1 python tools/ncu_step.py --config c4 --iters 0 > gpurun_out/ncu_ps_$1.log 2>&1
done
