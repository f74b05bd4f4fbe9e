mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > gpurun_out/cl_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/cl_tests.log
timeout 300 python tools/tts_ab.py 11 PERS_TMA=20000000 > gpurun_out/ab_cluster.log 2>&1
ECMG_LIB_PATH=$PWD/build/variants/libfull_nocluster.so timeout 300 python tools/tts_ab.py 11 PERS_TMA=20000000 >> gpurun_out/ab_cluster.log 2>&1
