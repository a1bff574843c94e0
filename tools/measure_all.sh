#!/bin/bash
# Every measurement DESIGN.md quotes, in one GPU round trip (run under gpurun from the repo root):
#   GPU parity tests, the default bench line + launch list + ncu capture (tools/gpu_check.sh),
#   the Newton / cfg4 / dense / cfg0-2 / reference bench lines, the cost constants C and C0,
#   and the sVELO experiment tables.  Results land in gpurun_out/ with the prefix $1 (default r1).
set -u
P=${1:-r1}
mkdir -p gpurun_out
bash tools/gpu_check.sh
run() {  # name, args...
    local name=$1
    shift
    timeout 900 python bench.py "$@" > gpurun_out/${P}_bench_${name}.json 2> gpurun_out/${P}_bench_${name}.err
}
run newton --update newton --steps 3 --no-cpu-baseline
run cfg4 --config cfg4 --events-per-rank 200 --steps 3 --no-cpu-baseline
run dense --dense --steps 2 --no-cpu-baseline --e2e-steps 1
for c in cfg0 cfg1 cfg2; do run $c --config $c --steps 5 --no-cpu-baseline; done
run ref --impl reference --steps 1 --warmup 0
timeout 600 python tools/cost_constants.py > gpurun_out/${P}_cost_constants_cfg3.json 2>&1
timeout 900 python tools/svelo_experiment.py --out gpurun_out/${P}_svelo_experiment > /dev/null 2>&1
python - "$P" <<'PY'
import json, sys
p = sys.argv[1]
for f in ("newton", "cfg4", "dense", "cfg0", "cfg1", "cfg2", "ref"):
    try:
        d = json.load(open(f"gpurun_out/{p}_bench_{f}.json"))
        print(f, "%.4g" % d["value"], round(d["ms_per_step"], 2), d.get("roofline", {}).get("frac"))
    except Exception as exc:  # report and go on: one failed line must not hide the others
        print(f, "FAILED", exc)
PY
