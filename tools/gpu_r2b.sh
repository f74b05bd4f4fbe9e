mkdir -p gpurun_out
timeout 900 python tools/diag_c4_rhs.py 7 > gpurun_out/diag_c4_rhs.log 2>&1; echo exit=$? >> gpurun_out/diag_c4_rhs.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_new.log 2>&1; echo exit=$? >> gpurun_out/bench_new.log
timeout 300 python bench.py --gpus 2 > gpurun_out/bench_gpus2.log 2>&1; echo exit=$? >> gpurun_out/bench_gpus2.log
