set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r4_pytest.txt
timeout 400 python bench.py > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
SMALL="python bench.py --events-per-rank 296 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$SMALL > gpurun_out/r4_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_launches.csv $SMALL > gpurun_out/r4_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"multistart|grid_separable" -s 4 -c 2 -o gpurun_out/r4_prof $SMALL > gpurun_out/r4_ncu2.log 2>&1
echo ncu_rc=$?
cat gpurun_out/r4_pytest.txt; cat gpurun_out/r4_bench.json
