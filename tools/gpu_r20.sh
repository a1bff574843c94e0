timeout 600 python -m pytest tests/test_svelo.py -m gpu -q 2>&1 | tail -5
timeout 900 python tools/svelo_experiment.py --events 20 > gpurun_out/r20_svelo.log 2>&1
tail -3 gpurun_out/r20_svelo.log
cat profiles/r1_svelo_experiment.md
mkdir -p gpurun_out/prof && cp profiles/r1_svelo_experiment.* gpurun_out/prof/ 2>/dev/null
