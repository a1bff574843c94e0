#!/usr/bin/env python
"""Benchmark of the Artificial Retina hot path on B200 (one process per GPU).

A step = one pass of the whole hot path over this rank's
event batch: grid response + peak finding (grid AR) and multi-start
fixed-step ascent + merging (Algorithm 1), then the one result gather.

Workload (default): BASELINE.json configs[3] ("Run-3-like batch"), 10,000 events per
rank with distinct event ids (weak scaling: per-GPU work fixed as N grows), 1024^2 grid,
8192 seeds x 50 iterations.  Metric: unit.hit evaluations/s (whole job), plus events/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import configs as C  # noqa: E402
from synth import events as G  # noqa: E402

METRIC = "retina unit·hit evaluations/s (events/s alongside)"
UNIT = "pairs/s"
MUFU_PER_SM_CLK = 16      # measured: tools/pipe_microbench (15.95 ex2/clk/SM)
FMA_PER_SM_CLK = 128      # measured: 121.5 FFMA/clk/SM; FFMA2 does not double it
N_SM = 148


def peaks_json():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p))
    return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0, "fallback": True}


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--events-per-rank", type=int, default=None)
    ap.add_argument("--chunk-events", type=int, default=1024)
    ap.add_argument("--grid-buffer-gb", type=float, default=5.0, help="device memory for the per-chunk response grids")
    ap.add_argument("--dense", action="store_true",
                    help="Z12 'dense' variant: every downstream plane hit (no acceptance cut), ~4,100 hits/event "
                         "for cfg3 as the config text states")
    ap.add_argument("--overlap-peaks", action="store_true",
                    help="peak scan of grid chunk c on a second stream while chunk c+1 is computed")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-events", type=int, default=3)
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="skip the CUDA-graph replay measurement")
    ap.add_argument("--update", default="gradient", choices=["gradient", "newton"],
                    help="multi-start update: BASELINE fixed-step ascent, or the paper's Truncated Newton")
    return ap.parse_args()


def make_spec(cfg):
    from paper_1709_08610_b200.pipeline import PathSpec
    return PathSpec(model=cfg.model, sigma=cfg.sigma, nodes=G.axis_nodes(cfg) if cfg.axes else [],
                    peak_threshold=cfg.peak_threshold, peak_capacity=cfg.peak_capacity, n_seeds=cfg.n_seeds,
                    n_iters=cfg.n_iters, step=cfg.step, box_lo=cfg.box_lo, box_hi=cfg.box_hi,
                    merge_radius=cfg.merge_radius, track_threshold=cfg.track_threshold,
                    track_capacity=cfg.track_capacity, z_ref=cfg.z_ref)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML every 100 ms while running."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - reported in the JSON
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(cfg, n_events: int):
    """The fp64 oracle, as it stands, on a bounded sample of the same workload: the full
    grid + peaks of `n_events` events and their full multi-start + merge."""
    from oracle import oracle as ora
    ev = list(range(n_events))
    b = G.make_batch(cfg, ev)
    seeds = G.make_seeds(cfg, ev)
    nodes = G.axis_nodes(cfg) if cfg.axes else []
    nh = float(b.n_hits)
    t0 = time.perf_counter()
    pairs = 0.0
    if nodes:
        g = ora.grid(cfg.model, b.offsets, b.hits, nodes, cfg.sigma)
        ora.peaks(g, cfg.P, cfg.peak_threshold, cfg.peak_capacity)
        pairs += nh * cfg.n_units
    if cfg.n_seeds:
        th, R, _ = ora.multistart(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, cfg.n_iters, cfg.step,
                                  cfg.box_lo, cfg.box_hi, want_grad=False)
        ora.merge(th, R, cfg.merge_radius, cfg.track_threshold, cfg.track_capacity)
        pairs += nh * cfg.n_seeds * (cfg.n_iters + 1)
    dt = time.perf_counter() - t0
    return {"value": pairs / dt, "unit": UNIT, "cores": ora.num_threads(), "kind": "oracle",
            "events_per_s": n_events / dt, "seconds": dt,
            "sample": f"{n_events} event(s) of {cfg.name}: full {'x'.join(str(a[2]) for a in cfg.axes)} grid + "
                      f"peaks and {cfg.n_seeds} seeds x {cfg.n_iters + 1} passes + merge; {pairs:.3e} pairs"}


def run_reference(a):
    rank, world, _ = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0 alone runs the oracle here, on all
    # the host's cores (read by OpenMP when the oracle library is first loaded, just below)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    cfg = C.get_config(a.config, dense=True) if a.dense else C.get_config(a.config)
    steps = []
    for _ in range(a.warmup + a.steps):
        steps.append(oracle_sample(cfg, a.cpu_sample_events))
    timed = steps[a.warmup:]
    value = statistics.median(s["value"] for s in timed)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.median(s["seconds"] for s in timed),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{cfg.name} (bounded sample, CPU oracle)",
                                            "events_per_step": a.cpu_sample_events},
            "events_per_s": statistics.median(s["events_per_s"] for s in timed),
            "cpu_baseline": {k: timed[-1][k] for k in ("kind", "cores", "sample")} | {"value": value, "unit": UNIT},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    a = args_()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    from paper_1709_08610_b200 import dist as D
    from paper_1709_08610_b200 import retina as RT
    from paper_1709_08610_b200.pipeline import PhaseTimer, RetinaPipeline, upload

    rank, world, local = D.env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    RT.lib()  # fail loudly if the native library is missing
    cfg = C.get_config(a.config, dense=True) if a.dense else C.get_config(a.config)
    E = a.events_per_rank or cfg.n_events
    ev_ids = range(rank * E, (rank + 1) * E)  # weak scaling: distinct events per rank
    t0 = time.perf_counter()
    batch = G.make_batch(cfg, ev_ids)
    seeds = G.make_seeds(cfg, ev_ids)
    gen_s = time.perf_counter() - t0
    spec = make_spec(cfg)
    if a.update == "newton":
        if cfg.model == C.LINE2D or not cfg.n_seeds:
            raise SystemExit(f"--update newton needs a SLOPE2/SLOPE3 config with seeds ({cfg.name} has none)")
        spec.newton = C.newton_schedule(cfg)
    pipe = RetinaPipeline(spec, E, chunk_events=a.chunk_events, overlap_peaks=a.overlap_peaks,
                          grid_bytes_budget=a.grid_buffer_gb * 1e9)
    stream = torch.cuda.current_stream()
    dbatch = upload(batch.offsets, batch.hits, seeds)
    if a.update == "newton":  # the pairs count comes from the kernel's per-seed evaluation counts
        pipe.run(dbatch, stream=stream)
        torch.cuda.synchronize()
    pairs_grid, pairs_ms = pipe.pairs(dbatch)
    keep = 64

    def step(b, timer=None, t_ms=0.0):
        pipe.run(b, stream=stream, timer=timer)
        buf = D.pack(pipe.peak_idx[:E], pipe.peak_val[:E], pipe.peak_cnt[:E], pipe.t_theta[:E], pipe.t_resp[:E],
                     pipe.t_size[:E], pipe.t_count[:E], keep,
                     [rank, rank * E, E, 0, 0, t_ms, pairs_grid / 1e9, pairs_ms / 1e9])
        return D.gather(buf, world)

    for _ in range(a.warmup):
        step(dbatch)
    torch.cuda.synchronize()
    timer = PhaseTimer(stream)
    pipe.launches = 0
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(a.steps):
            gathered = step(dbatch, timer)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = pipe.launches
    phase_ms = timer.totals_ms()
    phase_n = timer.counts()
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / a.steps

    # ---- the same hot path replayed from a CUDA graph (all kernel launches of one pass)
    graph_ms = None
    if a.graph:
        graph = pipe.capture(dbatch)
        graph.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(a.steps):
            graph.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1) / a.steps], device="cuda")
        if world > 1:
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        graph_ms = float(tg.item())
        del graph

    # ---- e2e through the public API with host buffers (pinned H2D + D2H inside the region)
    e2e_steps = a.e2e_steps if a.e2e_steps is not None else max(1, min(a.steps, 5))
    off_h = torch.from_numpy(batch.offsets).pin_memory()
    hits_h = torch.from_numpy(batch.hits).pin_memory()
    seeds_h = torch.from_numpy(seeds).pin_memory()
    res_h = torch.empty(gathered.shape, dtype=torch.float32).pin_memory()
    h2d = off_h.numel() * 4 + hits_h.numel() * 4 + seeds_h.numel() * 4
    d2h = res_h.numel() * 4
    # two device copies of the inputs: the H2D copy of step i+1 (copy stream) overlaps the
    # compute of step i; every step still moves its own inputs host -> device inside the region
    bufs = []
    for _ in range(2):
        d_off, d_hits, d_seeds = (torch.empty_like(x, device="cuda") for x in (off_h, hits_h, seeds_h))
        bufs.append((d_off, d_hits, d_seeds,
                     dbatch.__class__(offsets=d_off, hits=d_hits, seeds=d_seeds,
                                      max_event_hits=dbatch.max_event_hits,
                                      n_hits_per_event=dbatch.n_hits_per_event)))
    copy_stream = torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [None, None]

    def h2d_into(i):
        d_off, d_hits, d_seeds, _ = bufs[i % 2]
        with torch.cuda.stream(copy_stream):
            if done[i % 2] is not None:
                copy_stream.wait_event(done[i % 2])  # the step that last read this buffer is done
            d_off.copy_(off_h, non_blocking=True)
            d_hits.copy_(hits_h, non_blocking=True)
            d_seeds.copy_(seeds_h, non_blocking=True)
            ready[i % 2].record(copy_stream)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    copy_stream.wait_stream(stream)
    h2d_into(0)
    for i in range(e2e_steps):
        stream.wait_event(ready[i % 2])
        g2 = step(bufs[i % 2][3])
        done[i % 2] = torch.cuda.Event()
        done[i % 2].record(stream)
        if i + 1 < e2e_steps:
            h2d_into(i + 1)
        res_h.copy_(g2, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    t2 = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_ms_step = float(t2.item()) / e2e_steps

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of every hot kernel; the dominant one (largest share of the step) on top
    pk = peaks_json()
    fmax = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    clk = clocks.summary()
    traffic = {}
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof))
        except Exception:
            traffic = {}
    work = {"grid": pairs_grid, "multistart": pairs_ms}
    roofs = {}
    for ph in (k for k in phase_ms if k in work):
        n_launch = phase_n[ph] / a.steps
        avg_ms = phase_ms[ph] / phase_n[ph]
        per_launch = work[ph] / n_launch
        pairs_s = per_launch / (avg_ms * 1e-3)
        if ph == "grid" and cfg.model in (C.SLOPE2, C.SLOPE3):
            # tcgen05 fp16-split contraction (RETINA_GRID_AUTO = RETINA_GRID_TENSOR_F16): 2 algorithmic
            # flops per (unit, hit) pair, executed as 3 kind::f16 products (h.h, h.l, l.h); the
            # fp32-accurate tensor peak is the measured dense bf16/f16 peak / 3
            peak = float(pk.get("bf16_tflops", 1590.0)) * 1e12 / 3.0
            r = {"bound": "tensor",
                 "kernel": "grid_tensor16pp_kernel (persistent, tcgen05.mma cta_group::2 kind::f16, fp16 hi/lo split)",
                 "achieved": 2.0 * pairs_s / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                 "frac": 2.0 * pairs_s / peak,
                 "peak_basis": "MEASURED_PEAKS.json bf16_tflops (burst; f16 = bf16 rate) / 3 (three f16 products "
                               "per pair); algorithmic flops = 2 per unit.hit pair",
                 "executed_f16_frac": 6.0 * pairs_s / (peak * 3.0)}
        else:
            peak = N_SM * MUFU_PER_SM_CLK * fmax  # 1 MUFU.EX2 per pair
            kname = {"grid": "grid_separable/direct",
                     "multistart": "newton_kernel" if a.update == "newton" else "multistart_kernel"}[ph]
            r = {"bound": "alu", "kernel": kname,
                 "achieved": pairs_s / 1e9, "peak": peak / 1e9, "unit": "Gpair/s (1 MUFU.EX2 per pair)",
                 "frac": pairs_s / peak,
                 "peak_basis": f"{N_SM} SMs x {MUFU_PER_SM_CLK} MUFU.EX2/clk/SM (measured 15.95) x sm_max_mhz "
                               f"{fmax / 1e6:.0f} (MEASURED_PEAKS.json); the loop's 7 FMA-pipe lane-ops per pair make "
                               "the FMA pipe a co-limit (~14 pairs/clk/SM at the 97 lanes/clk measured for "
                               "FFMA2 with register operands, tools/pipe_microbench.cu)",
                 "frac_at_measured_clock": (pairs_s / (N_SM * MUFU_PER_SM_CLK * clk["sm_mhz"] * 1e6)
                                            if clk.get("sm_mhz") else None)}
        r.update({"launch_ms": avg_ms, "pairs_per_launch": per_launch, "pairs_per_s": pairs_s,
                  "share_of_step": phase_ms[ph] / a.steps / ms_step, "traffic": None})
        if ph == "multistart" and a.update == "newton":
            r["work_basis"] = ("pairs = sum over seeds of response evaluations (q Hessian-mode + line-search "
                               "trials + final; counted by the kernel, PAPER.md:200-201 cost unit) x event hits")
        if ph in traffic and not (ph == "multistart" and a.update == "newton"):
            r["traffic"] = traffic[ph]["dram_bytes_per_event"] * E / n_launch
            r["traffic_unit"] = "bytes/launch (ncu dram read+write per event x events per launch)"
        roofs[ph] = r
    dom = max(roofs, key=lambda k: roofs[k]["share_of_step"])
    roof = dict(roofs[dom])
    total_pairs = (pairs_grid + pairs_ms) * world
    line = {
        "metric": METRIC, "value": total_pairs / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "events_per_s": E * world / (ms_step * 1e-3),
        "config": {"workload": f"{cfg.name}{' dense (Z12: no acceptance cut)' if a.dense else ''}: "
                               f"BASELINE.json configs[{cfg.name[-1]}], {E} events per GPU "
                               f"(ids rank*{E}..), {'x'.join(str(x[2]) for x in cfg.axes)} "
                               f"{C.MODEL_NAME[cfg.model].upper()} grid + {'x'.join(['3'] * cfg.P)} peaks "
                               f"(R0={cfg.peak_threshold}) + sub-cell estimates, "
                               + (f"{cfg.n_seeds} seeds x {cfg.n_iters} fixed-step iterations + merge"
                                  if a.update == "gradient" else
                                  f"{cfg.n_seeds} seeds x q=3 Truncated-Newton steps (sigma schedule) + merge"),
                   "events_per_rank": E, "hits_per_event_mean": float(batch.n_hits) / E,
                   "pairs_grid_per_rank": pairs_grid, "pairs_multistart_per_rank": pairs_ms,
                   "l2": "inputs > L2 (hits %.0f MB, seeds %.0f MB, grid writes %.1f GB per step)" % (
                       batch.hits.nbytes / 1e6, seeds.nbytes / 1e6, 4.0 * cfg.n_units * E / 1e9),
                   "parallelism": f"dp{world} (events sharded, 1 all_gather of results)",
                   "arithmetic": ("fp32; the grid contraction as three fp16 tensor-core products of an exact "
                                  "hi/lo split of each fp32 factor, accumulated in fp32 (fp32-level accuracy, "
                                  "T1 1e-5)" if cfg.model in (C.SLOPE2, C.SLOPE3) else "fp32"),
                   "grid_chunk_events": pipe.chunk},
        "phases_ms_per_step": {k: v / a.steps for k, v in phase_ms.items()},
        "roofline": roof,
        "roofline_kernels": roofs,
        "clocks": clk,
        "e2e": {"value": total_pairs / (e2e_ms_step * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms_step},
        "gpu_launches": launches,
        "cuda_graph": (None if graph_ms is None else
                       {"ms_per_step_without_gather": graph_ms,
                        "value": (pairs_grid + pairs_ms) * world / (graph_ms * 1e-3),
                        "note": "the pass replayed from one captured CUDA graph (no result pack/gather)"}),
        "gen_seconds": gen_s,
    }
    if world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = oracle_sample(cfg, a.cpu_sample_events)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
