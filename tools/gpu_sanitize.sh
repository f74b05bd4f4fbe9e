# compute-sanitizer (memcheck, racecheck, synccheck) over every kernel family at 16^3 - 64^3 (tools/sanitize_run.py),
# the fp64 FMA peak microbenchmark and the fp64 op counts of k_rhs_c4 (its ALU roofline)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 ncu --clock-control none -k regex:k_rhs_c4 -c 1 --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --csv python tools/exp_timing.py 8 rhs > gpurun_out/ncu_rhs_flops.csv 2>&1
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo exit=$? >> gpurun_out/sanitizer_memcheck.log
timeout 1500 $CS --tool synccheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer_synccheck.log 2>&1; echo exit=$? >> gpurun_out/sanitizer_synccheck.log
timeout 2400 $CS --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_run.py small > gpurun_out/sanitizer_racecheck.log 2>&1; echo exit=$? >> gpurun_out/sanitizer_racecheck.log
