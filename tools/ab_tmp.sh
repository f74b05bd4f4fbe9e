mkdir -p gpurun_out
: > gpurun_out/ab_rhs.log
for v in default nof2f nof2f_zc64 zc64; do
  echo "== $v" >> gpurun_out/ab_rhs.log
  if [ $v = default ]; then timeout 300 python tools/exp_timing.py 8 rhs >> gpurun_out/ab_rhs.log 2>&1; timeout 300 python tools/tts_ab.py 9 PERS_TMA=20000000 >> gpurun_out/ab_rhs.log 2>&1;
  else ECMG_LIB_PATH=$PWD/build/variants/libfull_$v.so timeout 300 python tools/exp_timing.py 8 rhs >> gpurun_out/ab_rhs.log 2>&1; ECMG_LIB_PATH=$PWD/build/variants/libfull_$v.so timeout 300 python tools/tts_ab.py 9 PERS_TMA=20000000 >> gpurun_out/ab_rhs.log 2>&1; fi
done
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "rhs" > gpurun_out/rhs_test.log 2>&1
ECMG_LIB_PATH=$PWD/build/variants/libfull_nof2f.so python -c "
import sys; sys.path.insert(0,'.')
from paper_1506_02983_b200 import ecmg
" >> gpurun_out/rhs_test.log 2>&1
python tools/rhs_dump.py /tmp/b_def.npy >> gpurun_out/rhs_test.log 2>&1
ECMG_LIB_PATH=$PWD/build/variants/libfull_nof2f.so python tools/rhs_dump.py /tmp/b_nof2f.npy >> gpurun_out/rhs_test.log 2>&1
python -c "
import numpy as np
a=np.load('/tmp/b_def.npy'); b=np.load('/tmp/b_nof2f.npy')
print('max rel diff nof2f vs default', float(np.max(np.abs(a-b))/np.max(np.abs(a))))
" >> gpurun_out/rhs_test.log 2>&1
