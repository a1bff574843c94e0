timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r9_pytest.txt
timeout 400 python bench.py > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err
SMALL="python bench.py --events-per-rank 296 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$SMALL > gpurun_out/r9_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launches.csv $SMALL > gpurun_out/r9_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"multistart|grid_tensor" -s 4 -c 2 -o gpurun_out/r9_prof $SMALL > gpurun_out/r9_ncu2.log 2>&1
echo ncu_rc=$?
cat gpurun_out/r9_pytest.txt; python -c "
import json; d=json.load(open('gpurun_out/r9_bench.json')); print(d['value'], d['ms_per_step'], d['phases_ms_per_step']); print({k:(v['frac'],v['achieved'],v['unit']) for k,v in d['roofline_kernels'].items()}); print(d['clocks'], d['e2e'])"
