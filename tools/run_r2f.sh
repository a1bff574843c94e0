#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/f_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.txt 2>&1; echo "smoke rc $?" >> gpurun_out/f_smoke.txt
timeout 600 python bench.py --ms-algo culled --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_culled.json 2>/dev/null
timeout 600 python bench.py --ms-algo culled --grid-algo culled --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_culled_grid.json 2>/dev/null
timeout 600 python bench.py --config cfg2 --ms-algo culled --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_cfg2_culled.json 2>/dev/null
timeout 900 python bench.py --config cfg4 --ms-algo culled --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_cfg4full_culled.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"newton_kernel|multistart_culled" -s 4 -c 2 -o gpurun_out/f_prof_culled -f python tools/kbench.py --config cfg3 --events 296 --phases culled,newton_culled --reps 1 > gpurun_out/f_ncu.log 2>&1
echo done
