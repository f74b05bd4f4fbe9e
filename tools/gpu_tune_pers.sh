timeout 600 python tools/tune_persistent.py 300000 40000 5000 300000 40000 > gpurun_out/tune_pers.log 2>&1; echo exit=$? >> gpurun_out/tune_pers.log
timeout 400 python tools/run_c5.py 9 0 > gpurun_out/c5_run.log 2>&1; echo exit=$? >> gpurun_out/c5_run.log
