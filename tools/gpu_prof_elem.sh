timeout 300 python tools/ncu_step.py --config c3 --skip-run --iters 4 > gpurun_out/ncu_step_plain.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_elem --launch-skip 1 --launch-count 2 -o gpurun_out/p_elem python tools/ncu_step.py --config c3 --skip-run --iters 4 > gpurun_out/ncu_pe.log 2>&1
