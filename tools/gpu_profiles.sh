# profiles for the committed summaries: plain runs first (exit 0), then ncu (one GPU, single process).
# --launch-skip 3: INIT, K1, K2 of iteration 0 are skipped (iteration 0's K1 reads no p_old).
set -x
for c in c4 c3; do timeout 300 python tools/ncu_step.py --config $c --skip-run --iters 4 > gpurun_out/plain_$c.log 2>&1 || exit 1; done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_const_tma --launch-skip 3 --launch-count 2 -o gpurun_out/p_const python tools/ncu_step.py --config c4 --skip-run --iters 4 > gpurun_out/ncu_pc.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_jcg_elem_tma --launch-skip 3 --launch-count 2 -o gpurun_out/p_elem python tools/ncu_step.py --config c3 --skip-run --iters 4 > gpurun_out/ncu_pe.log 2>&1
for c in c4 c3; do
  timeout 300 python tools/ncu_step.py --config $c --iters 10 --host-loop > gpurun_out/run_$c.log 2>&1 || exit 1
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/ncu_step.py --config $c --iters 10 --host-loop > gpurun_out/ncu_l$c.log 2>&1
done
