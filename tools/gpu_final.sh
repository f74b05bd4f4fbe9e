# round-end evidence: default bench line (as the driver runs it), the reference arm, C3 bench, then the
# ncu captures (each after its plain run exited 0)
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo exit=$? >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo exit=$? >> gpurun_out/bench_reference.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo exit=$? >> gpurun_out/bench_c3.log
bash tools/gpu_profiles.sh
