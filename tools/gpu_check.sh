#!/bin/bash
# One GPU round trip (run under gpurun): GPU parity tests, the default bench line, the launch
# list and one ncu --set full capture of the hot kernels on a small bench, summarised into
# profiles/ (copied back through gpurun_out/).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
SMALL="python bench.py --events 296 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$SMALL > gpurun_out/small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL \
    > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"multistart|grid_tensor16pp" -s 4 -c 2 \
    -o gpurun_out/prof $SMALL > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/pytest_gpu.txt
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'], d['clocks'])"
