TTS_CFG=c3 timeout 300 python tools/tts_ab.py 7 PERS_TMA=3000000 PERS_TMA=20000000 > gpurun_out/ab_c3.log 2>&1
timeout 300 python tools/tts_ab.py 11 PERS_TMA=20000000 > gpurun_out/ab_c4_new.log 2>&1
