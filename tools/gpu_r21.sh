timeout 900 python tools/svelo_experiment.py --sweep --events 10 > gpurun_out/r21_sweep.log 2>&1
cat gpurun_out/r21_sweep.log | tail -8
mkdir -p gpurun_out/prof && cp profiles/r1_svelo_experiment_sweep.* gpurun_out/prof/ 2>/dev/null
