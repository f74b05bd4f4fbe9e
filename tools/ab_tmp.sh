mkdir -p gpurun_out
: > gpurun_out/ab_prio.log
for v in default prio_zc1 prio_zc4 zc1; do
  echo "== $v" >> gpurun_out/ab_prio.log
  if [ $v = default ]; then timeout 300 python tools/tts_ab.py 11 PERS_TMA=20000000 >> gpurun_out/ab_prio.log 2>&1;
  else ECMG_LIB_PATH=$PWD/build/variants/libfull_$v.so timeout 300 python tools/tts_ab.py 11 PERS_TMA=20000000 >> gpurun_out/ab_prio.log 2>&1; fi
done
