#!/usr/bin/env python
"""Benchmark of the Artificial Retina hot path on B200 (one process per GPU).

A step = one pass of the whole hot path over this rank's
event batch: grid response + peak finding + sub-cell estimates (grid AR) and
multi-start fixed-step ascent + merging (Algorithm 1), then the rank's result
record (retina_pack_results) and the one all_gather.

Workload (default): BASELINE.json configs[3] ("Run-3-like batch"): 10,000 events, 1024^2 grid,
8192 seeds x 50 iterations.  At N GPUs the SAME 10,000 events are sharded (strong scaling,
SURVEY.md §8(e): rank r owns [r E / N, (r + 1) E / N)); --scaling weak gives every rank its own
--events-per-rank events instead.  Metric: unit.hit evaluations/s (whole job), plus events/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scaling strong|weak]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

`--gpus N` without a torchrun environment launches the N ranks itself (torch.distributed.run,
127.0.0.1); NCCL's INIT log is left on (stderr) so the communicator lines show the N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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
FMA_REG_LANES = 97        # measured FMA-pipe lanes/clk/SM for FFMA2 with register operands (85-97)
N_SM = 148
# FMA-pipe lane-ops per (seed, hit) pair of the multi-start passes: fixed-step
# iterations (R not accumulated), Newton Hessian-mode and R-only evaluations
FMA_OPS = {"slope2_iter": 7, "slope3_iter": 8, "line2d_iter": 9, "hessian": 13, "r_only": 6}


def binding_pairs_per_clk(ops: float, fma_lanes: float = FMA_PER_SM_CLK) -> float:
    """Pairs/clk/SM of a loop with one MUFU.EX2 and `ops` FMA-pipe lane-ops per pair: the lower
    of the MUFU rate and the FMA pipe's rate (nominal 128 lanes/clk/SM; measured 121.5 for FFMA
    with immediate operands, 85-97 for FFMA2 with register operands, so loops near the FMA bound
    land below 1.0 of the nominal figure -- `fma_lanes` = FMA_REG_LANES gives the measured one)."""
    return min(MUFU_PER_SM_CLK, fma_lanes / ops)


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
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's batch sharded over the ranks (default); weak: --events-per-rank "
                         "events on every rank")
    ap.add_argument("--events", type=int, default=None, help="strong scaling: total events (default: the config's)")
    ap.add_argument("--events-per-rank", type=int, default=None, help="weak scaling: events per rank")
    ap.add_argument("--chunk-events", type=int, default=10000,
                    help="events per grid chunk (at most; chunks are equal; larger chunks keep the grid kernel "
                         "and the peak scan in full waves: cfg3 1,024 / 2,500 / 10,000 gave grid + peaks 50.4 / "
                         "48.9 / 47.8 ms per step)")
    ap.add_argument("--grid-buffer-gb", type=float, default=48.0,
                    help="device memory for the per-chunk response grids (cfg3: the whole 10,000-event batch, 42 GB; "
                         "cfg4: chunks of 500 events)")
    ap.add_argument("--dense", action="store_true",
                    help="Z12 'dense' variant: every downstream plane hit (no acceptance cut), ~4,100 hits/event "
                         "for cfg3 as the config text states")
    ap.add_argument("--overlap-peaks", action="store_true",
                    help="peak scan of grid chunk c on a second stream while chunk c+1 is computed")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-events", type=int, default=3, help="--impl reference: events per step")
    ap.add_argument("--cpu-plan", default="declared", choices=["declared", "quick"],
                    help="cpu_baseline sample: the SURVEY.md §8(d) declared subsample, or 1 event per phase (tests)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="skip the CUDA-graph replay measurement")
    ap.add_argument("--ms-algo", default="dense", choices=["dense", "culled"],
                    help="multi-start kernel (fixed step, or Newton with --update newton): dense (every pair, the metric's definition) or culled "
                         "(SLOPE2/SLOPE3: the same results bit for bit, evaluating only pairs whose weight can be "
                         "non-zero; value then counts the pairs actually evaluated)")
    ap.add_argument("--grid-algo", default="dense", choices=["dense", "culled"],
                    help="grid kernel: dense (every unit.hit pair) or culled (RETINA_GRID_TENSOR_F16_CULLED: each "
                         "tile contracts only the hits that can reach it; within T1 of the dense grid; value "
                         "then counts the pairs actually contracted)")
    ap.add_argument("--update", default="gradient", choices=["gradient", "newton"],
                    help="multi-start update: BASELINE fixed-step ascent, or the paper's Truncated Newton")
    ap.add_argument("--dist-check", action="store_true",
                    help="no GPU work: initialise the process group (gloo without CUDA), shard the batch, "
                         "all_gather each rank's event range and hit count, rank 0 prints them (launcher test)")
    return ap.parse_args()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(a):
    """`--gpus N` outside torchrun: launch N ranks with torch.distributed.run and return its exit
    code; inside torchrun the world size must equal --gpus.  Returns None when this process is a rank."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if a.gpus <= 1:
            return None
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        return subprocess.call(cmd, env=env)
    if int(ws) != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={ws}: launch one rank per GPU")
    return None


def rank_events(a, cfg, rank: int, world: int):
    """This rank's event ids and the scaling mode."""
    from paper_1709_08610_b200 import dist as D
    if a.scaling == "weak":
        E = a.events_per_rank or cfg.n_events
        return range(rank * E, (rank + 1) * E), "weak"
    n_total = a.events or cfg.n_events
    if n_total < world:  # single-event configs (cfg0, cfg1): replicas only
        return range(n_total), "replicas"
    return range(*D.shard(n_total, rank, world)), "strong"


def dist_check(a):
    import torch
    import torch.distributed as dist
    from paper_1709_08610_b200 import dist as D
    rank, world, _ = D.env()
    if world > 1:
        dist.init_process_group("gloo")
    cfg = C.get_config(a.config)
    ids, mode = rank_events(a, cfg, rank, world)
    b = G.make_batch(cfg, ids)
    mine = torch.tensor([rank, ids.start, ids.stop, b.n_hits], dtype=torch.int64)
    allr = [torch.zeros_like(mine) for _ in range(world)]
    if world > 1:
        dist.all_gather(allr, mine)
    else:
        allr = [mine]
    if rank == 0:
        print(json.dumps({"dist_check": True, "world": world, "scaling": mode,
                          "shards": [x.tolist() for x in allr]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


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
def _grid_plan(cfg, n_events, z_planes=None):
    nodes = G.axis_nodes(cfg)
    if z_planes is not None and cfg.P == 3:  # a bounded slab of the z0 axis (1-core cfg4 sample)
        nodes = nodes[:2] + [nodes[2][:z_planes]]
    return nodes


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


# SURVEY.md §8(d) "Oracle timing": declared subsamples (events for the grid phase, events for the
# multi-start phase) on all cores and on 1 core; cfg0-2 run in full on all cores.
CPU_PLAN = {"cfg0": ((1, 1), (1, 1, None)), "cfg1": ((1, 0), (1, 0, None)), "cfg2": ((0, 200), (0, 16, None)),
            "cfg3": ((16, 64), (1, 4, None)), "cfg4": ((2, 16), (1, 1, 16))}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_phases(cfg, grid_events: int, ms_events: int, threads: int, z_planes=None):
    """Times the oracle's grid+peaks phase and multi-start+merge phase on `threads` OpenMP threads."""
    from oracle import oracle as ora
    ora.set_num_threads(threads)
    out = {"threads": threads}
    if grid_events and cfg.axes:
        ev = list(range(grid_events))
        b = G.make_batch(cfg, ev)
        nodes = _grid_plan(cfg, grid_events, z_planes)
        cells = int(np.prod([len(n) for n in nodes]))
        t0 = time.perf_counter()
        g = ora.grid(cfg.model, b.offsets, b.hits, nodes, cfg.sigma)
        ora.peaks(g, cfg.P, cfg.peak_threshold, cfg.peak_capacity)
        dt = time.perf_counter() - t0
        pairs = float(b.n_hits) * cells
        out["grid"] = {"events": grid_events, "cells_per_event": cells, "pairs": pairs, "seconds": dt,
                       "pairs_per_s": pairs / dt, "pairs_per_s_per_core": pairs / dt / threads,
                       "seconds_per_full_event": dt / grid_events * cfg.n_units / cells}
    if ms_events and cfg.n_seeds:
        ev = list(range(ms_events))
        b = G.make_batch(cfg, ev)
        seeds = G.make_seeds(cfg, ev)
        t0 = time.perf_counter()
        th, R, _ = ora.multistart(cfg.model, b.offsets, b.hits, seeds, cfg.sigma, cfg.n_iters, cfg.step,
                                  cfg.box_lo, cfg.box_hi, want_grad=False)
        ora.merge(th, R, cfg.merge_radius, cfg.track_threshold, cfg.track_capacity)
        dt = time.perf_counter() - t0
        pairs = float(b.n_hits) * cfg.n_seeds * (cfg.n_iters + 1)
        out["multistart"] = {"events": ms_events, "pairs": pairs, "seconds": dt, "pairs_per_s": pairs / dt,
                             "pairs_per_s_per_core": pairs / dt / threads, "seconds_per_event": dt / ms_events}
    ph = [out[k] for k in ("grid", "multistart") if k in out]
    out["pairs_per_s"] = sum(p["pairs"] for p in ph) / sum(p["seconds"] for p in ph)
    # whole-config events/s extrapolated from the per-event phase times
    per_ev = (out["grid"]["seconds_per_full_event"] if "grid" in out else 0.0) + \
             (out["multistart"]["seconds_per_event"] if "multistart" in out else 0.0)
    out["events_per_s"] = 1.0 / per_ev
    return out


def cpu_baseline(cfg, plan: str = "declared"):
    all_cores = len(os.sched_getaffinity(0))
    (ga, ma), (g1, m1, zp) = CPU_PLAN.get(cfg.name, ((1, 1), (1, 1, None)))
    if plan == "quick":
        ga, ma, g1, m1, zp = min(ga, 1), min(ma, 1), 0, min(m1, 1), None
    full = oracle_phases(cfg, ga, ma, all_cores)
    one = oracle_phases(cfg, g1, m1, 1, z_planes=zp)
    desc = []
    if "grid" in full:
        desc.append(f"grid+peaks: {ga} full event(s) on {all_cores} threads, "
                    f"{g1} event(s){f' x {zp} z0 planes' if zp else ''} on 1")
    if "multistart" in full:
        desc.append(f"multi-start ({cfg.n_seeds} seeds x {cfg.n_iters + 1} passes) + merge: {ma} event(s) on "
                    f"{all_cores} threads, {m1} on 1")
    return {"value": full["pairs_per_s"], "unit": UNIT, "cores": all_cores, "kind": "oracle",
            "sample": f"{cfg.name} (SURVEY.md §8(d) declared subsample): " + "; ".join(desc),
            "cpu_model": cpu_model(), "events_per_s": full["events_per_s"], "all_cores": full, "one_core": one}


def run_reference(a):
    rank, world, _ = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0 alone runs the oracle here, on all
    # the host's cores (read by OpenMP when the oracle library is first loaded, just below)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    cfg = C.get_config(a.config, dense=True) if a.dense else C.get_config(a.config)
    from oracle import oracle as ora
    ora.set_num_threads(len(os.sched_getaffinity(0)))
    steps = []
    for _ in range(a.warmup + a.steps):
        steps.append(oracle_sample(cfg, a.cpu_sample_events))
    timed = steps[a.warmup:]
    value = statistics.median(s["value"] for s in timed)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.median(s["seconds"] for s in timed),
            "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{cfg.name} (bounded sample, CPU oracle)",
                                            "events_per_step": a.cpu_sample_events},
            "events_per_s": statistics.median(s["events_per_s"] for s in timed),
            "cpu_baseline": {k: timed[-1][k] for k in ("kind", "cores", "sample")} | {"value": value, "unit": UNIT,
                                                                                  "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    a = args_()
    if a.impl == "reference":
        return run_reference(a)
    rc = maybe_spawn(a)
    if rc is not None:
        sys.exit(rc)
    if a.dist_check:
        return dist_check(a)
    import torch
    import torch.distributed as dist

    from paper_1709_08610_b200 import dist as D
    from paper_1709_08610_b200 import retina as RT
    from paper_1709_08610_b200.pipeline import PhaseTimer, RetinaPipeline, upload

    rank, world, local = D.env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # communicator INIT lines (stderr) show the ranks
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    RT.lib()  # fail loudly if the native library is missing
    cfg = C.get_config(a.config, dense=True) if a.dense else C.get_config(a.config)
    ev_ids, scaling = rank_events(a, cfg, rank, world)
    E = len(ev_ids)
    t0 = time.perf_counter()
    batch = G.make_batch(cfg, ev_ids)
    seeds = G.make_seeds(cfg, ev_ids)
    gen_s = time.perf_counter() - t0
    spec = make_spec(cfg)
    if a.update == "newton":
        if cfg.model == C.LINE2D or not cfg.n_seeds:
            raise SystemExit(f"--update newton needs a SLOPE2/SLOPE3 config with seeds ({cfg.name} has none)")
        spec.newton = C.newton_schedule(cfg)
    if a.ms_algo == "culled":
        if cfg.model not in (C.SLOPE2, C.SLOPE3) or not cfg.n_seeds:
            raise SystemExit(f"--ms-algo culled needs a SLOPE2/SLOPE3 config with seeds ({cfg.name})")
        spec.ms_algorithm = RT.MS_CULLED
    if a.grid_algo == "culled":
        if cfg.model not in (C.SLOPE2, C.SLOPE3) or not cfg.axes:
            raise SystemExit(f"--grid-algo culled needs a SLOPE2/SLOPE3 grid config ({cfg.name})")
        spec.grid_algorithm = RT.GRID_TENSOR_F16_CULLED
    pipe = RetinaPipeline(spec, E, chunk_events=a.chunk_events, overlap_peaks=a.overlap_peaks,
                          grid_bytes_budget=a.grid_buffer_gb * 1e9)
    stream = torch.cuda.current_stream()
    dbatch = upload(batch.offsets, batch.hits, seeds)
    if a.update == "newton" or pipe.pairs_ev is not None or pipe.grid_pairs_ev is not None:
        # the pairs count comes from the kernel: per-seed evaluation counts (Newton) or the pairs
        # the culled kernel evaluated (one counted run, outside the timed region)
        pipe.count_pairs = pipe.pairs_ev is not None or pipe.grid_pairs_ev is not None
        pipe.run(dbatch, stream=stream)
        torch.cuda.synchronize()
        pipe.count_pairs = False
    pairs_grid, pairs_ms = pipe.pairs(dbatch)
    keep = 64
    hdr = D.header_words(rank, ev_ids.start, E, pairs_grid, pairs_ms)
    pack_out = torch.empty((RT.PACK_HEADER + E * D.record_width(spec.P, keep),), dtype=torch.int32, device="cuda")

    def step(b, timer=None):
        pipe.run(b, stream=stream, timer=timer)
        # the rank's result record, written on the device (retina_pack_results), then THE gather
        buf = D.pack(pipe.peak_idx[:E], pipe.peak_val[:E], pipe.peak_cnt[:E], pipe.t_theta[:E], pipe.t_resp[:E],
                     pipe.t_size[:E], pipe.t_count[:E], keep, hdr, out=pack_out, stream=stream)
        pipe.launches += 2
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
            timer.next_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = pipe.launches
    per_step = timer.per_step_ms()
    phase_med = {k: statistics.median(v) for k, v in per_step.items()}
    phase_n = timer.counts()

    # ---- per-rank timings and work, gathered once after the timed region; the step time is the max
    mine = torch.tensor([float(rank), float(E), ms, pairs_grid, pairs_ms]
                        + [phase_med.get(k, 0.0) for k in ("grid", "peaks", "multistart", "merge")],
                        dtype=torch.float64, device="cuda")
    ranks = [mine]
    if world > 1:
        ranks = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(ranks, mine)
    ranks = [r.cpu().tolist() for r in ranks]
    ms_max = max(r[2] for r in ranks)
    ms_step = ms_max / a.steps
    pairs_all = sum(r[3] + r[4] for r in ranks)
    events_all = sum(r[1] for r in ranks)

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
    res_h = torch.empty(gathered.shape, dtype=gathered.dtype).pin_memory()
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
    # the gathered records decode to every rank's event range (checked on rank 0)
    dec = D.unpack(gathered.cpu().numpy(), spec.P, keep)

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
    for ph in (k for k in phase_med if k in work):
        n_launch = phase_n[ph] / a.steps
        avg_ms = phase_med[ph] / n_launch
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
                     "multistart": ("newton_kernel" + (" (culled)" if a.ms_algo == "culled" else ""))
                     if a.update == "newton" else "multistart_kernel"}[ph]
            r = {"bound": "alu", "kernel": kname,
                 "achieved": pairs_s / 1e9, "peak": peak / 1e9, "unit": "Gpair/s (1 MUFU.EX2 per pair)",
                 "frac": pairs_s / peak,
                 "peak_basis": f"{N_SM} SMs x {MUFU_PER_SM_CLK} MUFU.EX2/clk/SM (measured 15.95) x sm_max_mhz "
                               f"{fmax / 1e6:.0f} (MEASURED_PEAKS.json); the loop's 7 FMA-pipe lane-ops per pair make "
                               "the FMA pipe a co-limit (~14 pairs/clk/SM at the 97 lanes/clk measured for "
                               "FFMA2 with register operands, tools/pipe_microbench.cu)",
                 "frac_at_measured_clock": (pairs_s / (N_SM * MUFU_PER_SM_CLK * clk["sm_mhz"] * 1e6)
                                            if clk.get("sm_mhz") else None)}
        if ph == "multistart":
            # the binding pipe of the loop: MUFU or the FMA pipe at its measured register-operand rate
            if a.update == "newton":
                q = len(spec.newton[0])
                # response evaluations per seed (the kernel's counts; the culled kernel's pairs are not
                # evaluations x hits)
                ev_mean = float(pipe.evals[:E].to(torch.float64).mean().item())
                cyc = (q / binding_pairs_per_clk(FMA_OPS["hessian"])
                       + max(0.0, ev_mean - q) / binding_pairs_per_clk(FMA_OPS["r_only"])) / ev_mean
                cyc_m = (q / binding_pairs_per_clk(FMA_OPS["hessian"], FMA_REG_LANES)
                         + max(0.0, ev_mean - q) / binding_pairs_per_clk(FMA_OPS["r_only"], FMA_REG_LANES)) / ev_mean
                basis = (f"{q} Hessian-mode evaluations (13 FMA-pipe lane-ops/pair) and {ev_mean - q:.2f} R-only "
                         f"evaluations (6) per seed on average")
            else:
                ops = FMA_OPS[{C.SLOPE2: "slope2_iter", C.SLOPE3: "slope3_iter"}.get(cfg.model, "line2d_iter")]
                cyc = 1.0 / binding_pairs_per_clk(ops)
                cyc_m = 1.0 / binding_pairs_per_clk(ops, FMA_REG_LANES)
                basis = f"{ops} FMA-pipe lane-ops per pair in the iterations"
            bpeak = N_SM * fmax / cyc
            bpeak_m = N_SM * fmax / cyc_m
            r["binding"] = {"peak_pairs_per_s": bpeak, "frac": pairs_s / bpeak,
                            "measured_fma_peak_pairs_per_s": bpeak_m, "frac_at_measured_fma": pairs_s / bpeak_m,
                            "basis": basis + f"; FMA pipe at its nominal {FMA_PER_SM_CLK} lanes/clk/SM (measured "
                                             f"{FMA_REG_LANES} for FFMA2 with register operands, tools/pipe_microbench.cu), "
                                             "MUFU at 16/clk/SM: the lower rate binds"}
        r.update({"launch_ms": avg_ms, "pairs_per_launch": per_launch, "pairs_per_s": pairs_s,
                  "share_of_step": phase_med[ph] / ms_step, "traffic": None,
                  "timing": f"median over {a.steps} steps of the phase's CUDA-event time per step"})
        if ph == "multistart" and a.ms_algo == "culled" and a.update == "gradient":
            r["kernel"] = "multistart_culled_kernel"
            r["work_basis"] = ("pairs = (seed, hit) pairs the culled kernel evaluated (counted on the device); "
                               "the skipped pairs have weight exactly +0")
        if ph == "multistart" and a.update == "newton" and a.ms_algo == "culled":
            r["work_basis"] = ("pairs = (seed, hit) pairs the culled Newton kernel's passes visited (counted on the "
                               "device, speculative line-search halvings included); the skipped pairs have weight "
                               "exactly +0")
        elif ph == "multistart" and a.update == "newton":
            r["work_basis"] = ("pairs = sum over seeds of response evaluations (q Hessian-mode + line-search "
                               "trials + final; counted by the kernel, PAPER.md:200-201 cost unit) x event hits")
        tcfg = traffic.get(cfg.name, {}) if not a.dense else {}  # per config: the capture's workload
        if ph in tcfg and not (ph == "multistart" and (a.update == "newton" or a.ms_algo == "culled")):
            r["traffic"] = tcfg[ph]["dram_bytes_per_event"] * E / n_launch
            r["traffic_unit"] = "bytes/launch (ncu dram read+write per event x events per launch)"
        roofs[ph] = r
    dom = max(roofs, key=lambda k: roofs[k]["share_of_step"])
    roof = dict(roofs[dom])
    n_total = a.events or cfg.n_events
    workload = (f"{cfg.name}{' dense (Z12: no acceptance cut)' if a.dense else ''}: BASELINE.json configs[{cfg.name[-1]}], "
                + (f"{n_total} events sharded over {world} GPU(s)" if scaling == "strong" else
                   f"{E} events per GPU (ids rank*{E}..)" if scaling == "weak" else
                   f"{E} event(s) replicated on each of {world} GPU(s)")
                + (f", {'x'.join(str(x[2]) for x in cfg.axes)} {C.MODEL_NAME[cfg.model].upper()} grid + "
                   f"{'x'.join(['3'] * cfg.P)} peaks (R0={cfg.peak_threshold}) + sub-cell estimates" if cfg.axes else "")
                + ((", " + (f"{cfg.n_seeds} seeds x {cfg.n_iters} fixed-step iterations + merge"
                            + (" (culled multi-start kernel: bit-identical results, pairs = pairs evaluated)"
                               if a.ms_algo == "culled" else "")
                            if a.update == "gradient" else
                            f"{cfg.n_seeds} seeds x q=3 Truncated-Newton steps (sigma schedule) + merge"
                            + (" (culled Newton kernel: bit-identical results, pairs = pairs visited)"
                               if a.ms_algo == "culled" else "")))
                   if cfg.n_seeds else ""))
    line = {
        "metric": METRIC, "value": pairs_all / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "events_per_s": events_all / (ms_step * 1e-3),
        "config": {"workload": workload,
                   "events_total": int(events_all), "events_per_rank": [int(r[1]) for r in ranks],
                   "hits_per_event_mean": float(batch.n_hits) / max(E, 1),
                   "pairs_grid_per_rank": pairs_grid, "pairs_multistart_per_rank": pairs_ms,
                   "l2": "inputs > L2 (hits %.0f MB, seeds %.0f MB, grid writes %.1f GB per step per rank)" % (
                       batch.hits.nbytes / 1e6, seeds.nbytes / 1e6, 4.0 * cfg.n_units * E / 1e9),
                   "parallelism": f"dp{world} (events sharded, 1 all_gather of device-packed results)",
                   "arithmetic": ("fp32; the grid contraction as three fp16 tensor-core products of an exact "
                                  "hi/lo split of each fp32 factor, accumulated in fp32 (fp32-level accuracy, "
                                  "T1 1e-5)" if cfg.model in (C.SLOPE2, C.SLOPE3) else "fp32"),
                   "grid_chunk_events": pipe.chunk},
        "phases_ms_per_step": phase_med,
        "phases_ms_per_step_all_steps": per_step,
        "per_rank": [{"rank": int(r[0]), "events": int(r[1]), "ms_per_step": r[2] / a.steps,
                      "pairs": r[3] + r[4], "phases_ms": dict(zip(("grid", "peaks", "multistart", "merge"), r[5:]))}
                     for r in ranks],
        "gathered": {"ranks": [d["rank"] for d in dec], "event_base": [d["event_base"] for d in dec],
                     "peaks_total": sum(d["peaks_total"] for d in dec),
                     "tracks_total": sum(d["tracks_total"] for d in dec),
                     "record_bytes_per_rank": int(pack_out.numel() * 4)},
        "roofline": roof,
        "roofline_kernels": roofs,
        "clocks": clk,
        "e2e": {"value": pairs_all / (e2e_ms_step * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms_step},
        "gpu_launches": launches,
        "cuda_graph": (None if graph_ms is None else
                       {"ms_per_step_without_gather": graph_ms,
                        "value": (pairs_grid + pairs_ms) * world / (graph_ms * 1e-3),
                        "note": "the pass replayed from one captured CUDA graph (no result pack/gather)"}),
        "gen_seconds": gen_s,
    }
    if world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, a.cpu_plan)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
