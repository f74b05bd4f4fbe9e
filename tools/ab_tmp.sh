mkdir -p gpurun_out
timeout 300 python tools/tts_ab.py 11 PERS_TMA=20000000,PERSISTENT=40000 PERS_TMA=20000000,PERSISTENT=300000 > gpurun_out/ab_persist.log 2>&1
TTS_CFG=c3 timeout 300 python tools/tts_ab.py 5 PERS_TMA=20000000,PERSISTENT=40000 PERS_TMA=20000000,PERSISTENT=300000 >> gpurun_out/ab_persist.log 2>&1
