rm -f gpurun_out/exptune.log
for c in 32 8 16 64 32; do echo "cchunk=$c" >> gpurun_out/exptune.log; ECMG_TUNE_EXP_TRUE_CHUNK=$c timeout 120 python tools/exp_timing.py 8 rich >> gpurun_out/exptune.log 2>&1; done
for l in 0 1 2 4 8; do echo "lchunk=$l" >> gpurun_out/exptune.log; ECMG_TUNE_EXP_LCHUNK=$l timeout 120 python tools/exp_timing.py 8 run >> gpurun_out/exptune.log 2>&1; done
