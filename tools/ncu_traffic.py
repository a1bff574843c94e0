#!/usr/bin/env python
"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per event of the grid and multi-start
kernels, from ncu --set full summaries (tools/ncu_summary.py JSON) of bench.py launches.

    python tools/ncu_traffic.py cfg3:profiles/r2_ncu_cfg3.json:296 cfg4:profiles/r2_ncu_cfg4.json:24

Each argument is config:summary:events-per-launch of the captured bench run; bench.py reports
`traffic` = bytes per event x events per launch for the matching config (null otherwise).
"""
import json
import os
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def nbytes(v: str) -> float:
    num, unit = v.split()
    return float(num) * UNIT[unit]


def main():
    out = {"source": "ncu --set full captures of bench.py launches (tools/ncu_summary.py JSON): "
                     "(dram__bytes_read.sum + dram__bytes_write.sum) per launch / events in that launch"}
    for arg in sys.argv[1:]:
        cfg, path, events = arg.split(":")
        events = int(events)
        ent = {}
        for k in json.load(open(path))["kernels"]:
            name = k["kernel"]
            phase = "grid" if "grid_tensor" in name else "multistart" if "multistart" in name else None
            if phase is None or phase in ent:
                continue
            b = nbytes(k["dram__bytes_read.sum"]) + nbytes(k["dram__bytes_write.sum"])
            ent[phase] = {"dram_bytes_per_event": b / events, "launch_events": events, "kernel": name,
                          "summary": os.path.relpath(path)}
        out[cfg] = ent
    json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                     "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
