CMD="python tools/variant_bench.py --config cfg4 --events 20 --reps 1"
$CMD > gpurun_out/r18_plain.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:multistart -s 1 -c 1 -o gpurun_out/r18_prof $CMD > gpurun_out/r18_ncu.log 2>&1
echo rc=$?
