# element-path profile (C3 256^3): plain run first, then one ncu --set full capture of K1 and K2, and
# the launch list (durations) of one full C3 ecmg_run
timeout 300 python tools/ncu_step.py --config c3 --skip-run --iters 4 > gpurun_out/ncu_step_plain.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_elem_tma --launch-skip 1 --launch-count 2 -o gpurun_out/p_elem python tools/ncu_step.py --config c3 --skip-run --iters 4 > gpurun_out/ncu_pe.log 2>&1
timeout 300 python tools/ncu_step.py --config c3 --iters 0 > gpurun_out/ncu_step_run.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/ncu_step.py --config c3 --iters 0 > gpurun_out/ncu_lc3.log 2>&1
