#!/bin/bash
# Round-2 measurement set in one GPU round trip (run under gpurun from the repo root); results in
# gpurun_out/ with prefix $1 (default r2): GPU parity suite (PARITY-STATS lines kept), the default
# bench line, the launch list of a 296-event bench and one ncu --set full capture of the hot kernels
# (cfg3 multistart + grid, cfg4 grid + 3x3x3 peaks + SLOPE3 multistart), and the other bench lines.
set -u
P=${1:-r2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/${P}_pytest_gpu_full.txt 2>&1
grep -E "PARITY-STATS|passed|failed" gpurun_out/${P}_pytest_gpu_full.txt > gpurun_out/${P}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
SMALL="python bench.py --events 296 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph"
$SMALL > gpurun_out/${P}_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches.csv $SMALL \
    > gpurun_out/${P}_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"multistart|grid_tensor16pp" -s 4 -c 2 \
    -o gpurun_out/${P}_prof_cfg3 $SMALL > gpurun_out/${P}_ncu_full.log 2>&1
SMALL4="python bench.py --config cfg4 --events 24 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-graph"
$SMALL4 > gpurun_out/${P}_small4.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_cfg4.csv $SMALL4 \
    > gpurun_out/${P}_ncu_launches4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"multistart|grid_tensor16pp|peaks3_brick" -s 6 -c 3 \
    -o gpurun_out/${P}_prof_cfg4 $SMALL4 > gpurun_out/${P}_ncu_full4.log 2>&1
echo "ncu rc=$?"
run() {  # name, args...
    local name=$1
    shift
    timeout 900 python bench.py "$@" > gpurun_out/${P}_bench_${name}.json 2> gpurun_out/${P}_bench_${name}.err
}
run newton --update newton --steps 5 --no-cpu-baseline
run cfg4 --config cfg4 --events 200 --steps 5 --no-cpu-baseline
run cfg4full --config cfg4 --steps 3 --warmup 3 --cpu-plan quick
run dense --dense --events 2000 --steps 3 --no-cpu-baseline --e2e-steps 1
run cfg4dense --config cfg4 --dense --events 100 --steps 3 --no-cpu-baseline --e2e-steps 1
for c in cfg0 cfg1 cfg2; do run $c --config $c --steps 5; done
run ref --impl reference --steps 1 --warmup 0
# the opt-in culled kernels (K4c / K6c bit-identical to K4 / K6; the culled grid within T1)
run culled --ms-algo culled --steps 5 --no-cpu-baseline
run culled_grid_and_ms --ms-algo culled --grid-algo culled --steps 5 --no-cpu-baseline
run cfg2_culled --config cfg2 --ms-algo culled --steps 5 --no-cpu-baseline
run cfg4full_culled --config cfg4 --ms-algo culled --steps 3 --warmup 3 --no-cpu-baseline
run newton_culled --update newton --ms-algo culled --steps 5 --no-cpu-baseline
run newton_culled_grid --update newton --ms-algo culled --grid-algo culled --steps 5 --no-cpu-baseline
timeout 600 python tools/cost_constants.py > gpurun_out/${P}_cost_constants_cfg3.json 2>&1
tail -2 gpurun_out/${P}_pytest_gpu.txt
python - "$P" <<'PY'
import json, sys
p = sys.argv[1]
for f in ("", "_newton", "_cfg4", "_cfg4full", "_dense", "_cfg4dense", "_cfg0", "_cfg1", "_cfg2", "_ref", "_culled",
          "_culled_grid_and_ms", "_cfg2_culled", "_cfg4full_culled", "_newton_culled", "_newton_culled_grid"):
    try:
        d = json.load(open(f"gpurun_out/{p}_bench{f}.json"))
        print(f or "default", "%.4g" % d["value"], round(d["ms_per_step"], 2), d.get("roofline", {}).get("frac"),
              round(d.get("events_per_s", 0)),
              {k: round(v, 2) for k, v in d.get("phases_ms_per_step", {}).items()})
    except Exception as exc:  # report and go on: one failed line must not hide the others
        print(f, "FAILED", exc)
PY
# repeatability: the default bench twice more on the same box
for k in 2 3; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${P}_bench_rep$k.json 2>/dev/null; done
python - "$P" <<'PY'
import json, sys
p = sys.argv[1]
for f in ("", "_rep2", "_rep3"):
    try:
        d = json.load(open(f"gpurun_out/{p}_bench{f}.json"))
        print("repeat", f or "_rep1", round(d["ms_per_step"], 2), round(d["roofline"]["frac"], 4))
    except Exception as exc:
        print(f, "FAILED", exc)
PY
