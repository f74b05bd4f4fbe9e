rm -f gpurun_out/tune_elem.log
timeout 200 python tools/tune_elem.py --zc paper_1506_02983_b200/libecmg.so c4_256 0 32 0 >> gpurun_out/tune_elem.log 2>&1
timeout 200 python tools/tune_elem.py --zc paper_1506_02983_b200/libecmg.so c4 0 >> gpurun_out/tune_elem.log 2>&1
timeout 200 python tools/tune_elem.py --zc paper_1506_02983_b200/libecmg.so c3 0 >> gpurun_out/tune_elem.log 2>&1
timeout 400 python tools/tune_elem.py --zc paper_1506_02983_b200/libecmg.so c5 0 >> gpurun_out/tune_elem.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo exit=$? >> gpurun_out/bench_c3.log
