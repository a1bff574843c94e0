"""One GPU's pass of the whole hot path over an event batch.

    S-A  grid AR (steps ii-iv):  retina_grid_response -> retina_find_peaks
                                                   -> retina_estimate_peaks
    S-B  Algorithm 1:            retina_multistart_optimize -> retina_merge_tracks

All arithmetic runs in libretina.so; this module only owns device buffers, slices the
CSR batch into chunks (the response grid of a chunk is produced, scanned for peaks and
then overwritten by the next chunk, so a 10,000-event batch needs ~1 GB of grid buffer,
not 42 GB), and counts the algorithmic work (unit.hit pairs) for the report.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence

import numpy as np
import torch

from . import retina as R


@dataclasses.dataclass
class PathSpec:
    """Hot-path parameters (the ABI arguments; see include/retina.h)."""
    model: int
    sigma: float
    nodes: Sequence[np.ndarray]          # fp32 node tables (grid path)
    peak_threshold: float
    peak_capacity: int
    n_seeds: int
    n_iters: int
    step: float
    box_lo: Sequence[float]
    box_hi: Sequence[float]
    merge_radius: Sequence[float]
    track_threshold: float
    track_capacity: int
    z_ref: float = 0.0
    sigma_ms: Optional[float] = None     # multi-start sigma (defaults to sigma)
    newton: Optional[tuple] = None       # (sigmas, etas, final_sigma, max_halvings): Newton update
    ms_algorithm: int = 0                # R.MS_DENSE, or R.MS_CULLED (SLOPE2/3: same results, fewer pairs)
    grid_algorithm: int = 0              # R.GRID_AUTO, or e.g. R.GRID_TENSOR_F16_CULLED

    @property
    def P(self) -> int:
        return R.MODEL_P[self.model]

    @property
    def cells(self) -> int:
        return int(np.prod([len(n) for n in self.nodes])) if self.nodes else 0


@dataclasses.dataclass
class DeviceBatch:
    offsets: torch.Tensor      # int32 [E+1] device
    hits: torch.Tensor         # fp32 [N, 4] device
    seeds: torch.Tensor        # fp32 [E, S, P] device
    max_event_hits: int
    n_hits_per_event: np.ndarray  # host int64 [E]

    @property
    def n_events(self) -> int:
        return self.offsets.numel() - 1


class RetinaPipeline:
    def __init__(self, spec: PathSpec, max_events: int, chunk_events: int = 256, device="cuda",
                 grid_bytes_budget: float = 2e9, overlap_peaks: bool = False):
        self.spec = spec
        self.device = torch.device(device)
        cells = spec.cells
        if cells:
            chunk_events = max(1, min(chunk_events, int(grid_bytes_budget // (4 * cells))))
        # equal chunks (a short last chunk leaves most of the GPU idle in its grid and peak scan)
        n_chunks = -(-max(1, max_events) // max(1, chunk_events))
        self.chunk = -(-max(1, max_events) // n_chunks)
        self.nodes = [torch.from_numpy(np.ascontiguousarray(n, np.float32)).to(self.device) for n in spec.nodes]
        shape = R.grid_shape(self.chunk, [len(n) for n in spec.nodes])[1:]  # (n2,) n0, n1: z0 planes outermost
        self.grid_buf = torch.empty((self.chunk,) + shape, dtype=torch.float32, device=self.device) if cells else None
        # With several chunks, the peak scan of chunk c (HBM-bound, small CTAs) runs on a second,
        # higher-priority stream while the tensor-core grid kernel computes chunk c+1 into a second
        # buffer: the two kernels co-reside on the SMs (the grid CTA leaves registers and threads free).
        self.overlap = bool(cells) and overlap_peaks and max_events > self.chunk
        self.grid_bufs = [self.grid_buf]
        self.side = None
        if self.overlap:
            self.grid_bufs.append(torch.empty_like(self.grid_buf))
            self.side = torch.cuda.Stream(self.device, priority=-1)
        # the many-CTA peak finder (slabs of 131,072 cells, or 3x3x3 plane blocks): one CTA per
        # event leaves the last wave of a chunk part-empty (cfg3, 2,048 events: 2.50 ms one CTA per
        # event, 2.20 ms in slabs; the dense-hit variant 5.14 vs 4.52)
        self.peak_ws = None
        if cells:
            ws = R.find_peaks_workspace_size(self.chunk, shape)
            self.peak_ws = torch.empty((max(ws, 4) // 4,), dtype=torch.int32, device=self.device)
        E, P = max_events, spec.P
        self.peak_idx = torch.empty((E, spec.peak_capacity), dtype=torch.int32, device=self.device)
        self.peak_val = torch.empty((E, spec.peak_capacity), dtype=torch.float32, device=self.device)
        # counts start at zero: a config without a grid (or without seeds) reports no peaks (tracks)
        self.peak_cnt = torch.zeros((E,), dtype=torch.int32, device=self.device)
        self.peak_theta = torch.empty((E, spec.peak_capacity, spec.P), dtype=torch.float32, device=self.device)
        S = spec.n_seeds
        self.theta = torch.empty((E, S, P), dtype=torch.float32, device=self.device)
        self.resp = torch.empty((E, S), dtype=torch.float32, device=self.device)
        # Newton path: response evaluations per seed (the paper's cost unit), counted by the kernel
        self.evals = torch.empty((E, S), dtype=torch.int32, device=self.device) if spec.newton is not None else None
        # culled multi-start (fixed step or Newton): the per-event seed permutation (workspace) and the
        # evaluated-pair count
        self.ms_ws = self.pairs_ev = None
        if spec.ms_algorithm == R.MS_CULLED and S:
            nb = R.multistart_workspace_size(E, S, spec.ms_algorithm)
            self.ms_ws = torch.empty((max(nb, 4) // 4,), dtype=torch.int32, device=self.device)
            self.pairs_ev = torch.zeros((1,), dtype=torch.int64, device=self.device)
        # culled grid: the pairs the tiles contracted
        self.grid_pairs_ev = None
        if spec.cells and spec.grid_algorithm == R.GRID_TENSOR_F16_CULLED:
            self.grid_pairs_ev = torch.zeros((1,), dtype=torch.int64, device=self.device)
        self.count_pairs = False  # run(): add the pairs the culled kernels evaluate to pairs_ev / grid_pairs_ev
        self.t_theta = torch.empty((E, spec.track_capacity, P), dtype=torch.float32, device=self.device)
        self.t_resp = torch.empty((E, spec.track_capacity), dtype=torch.float32, device=self.device)
        self.t_seed = torch.empty((E, spec.track_capacity), dtype=torch.int32, device=self.device)
        self.t_size = torch.empty((E, spec.track_capacity), dtype=torch.int32, device=self.device)
        self.t_count = torch.zeros((E,), dtype=torch.int32, device=self.device)
        self.launches = 0

    # ------------------------------------------------------------------ accounting
    def pairs(self, batch: DeviceBatch):
        """Algorithmic unit.hit pairs: grid = N_e x cells, multi-start = N_e x S x (n_iters+1);
        for the Newton update, N_e x (response evaluations of the event's seeds), read from the
        kernel's per-seed counts of the last pass (call after one run())."""
        n = batch.n_hits_per_event.astype(np.float64)
        grid = float(n.sum()) * self.spec.cells
        if self.grid_pairs_ev is not None:  # the pairs the culled grid contracted in the counted run
            grid = float(self.grid_pairs_ev.item())
        if self.pairs_ev is not None:  # the pairs the culled kernel evaluated in the counted run
            return grid, float(self.pairs_ev.item())
        if self.spec.newton is not None:
            E = batch.n_events
            ev = self.evals[:E].to(torch.float64).sum(dim=1).cpu().numpy()
            return grid, float((n * ev).sum())
        ms = float(n.sum()) * self.spec.n_seeds * (self.spec.n_iters + 1)
        return grid, ms

    def events_view(self, batch: DeviceBatch, e0: int, e1: int) -> R.Events:
        return R.Events(batch.offsets[e0:e1 + 1], batch.hits, self.spec.z_ref, batch.max_event_hits)

    # ------------------------------------------------------------------ the two paths
    def run_grid(self, batch: DeviceBatch, stream=None, timer=None):
        sp = self.spec
        E = batch.n_events
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        side = self.side if self.overlap else main
        if side is not main:
            side.wait_stream(main)
        freed = [None] * len(self.grid_bufs)  # event: the peak scan of the buffer's last chunk is done
        for ci, e0 in enumerate(range(0, E, self.chunk)):
            e1 = min(E, e0 + self.chunk)
            b = ci % len(self.grid_bufs)
            if freed[b] is not None:
                main.wait_event(freed[b])
            ev = self.events_view(batch, e0, e1)
            out = self.grid_bufs[b][: e1 - e0]
            if timer is not None:
                timer.start("grid", main)
            R.retina_grid_response(ev, sp.model, sp.sigma, self.nodes, out=out, stream=main,
                                   algorithm=sp.grid_algorithm,
                                   pairs_evaluated=self.grid_pairs_ev if self.count_pairs else None)
            if timer is not None:
                timer.stop("grid", main)
            if side is not main:
                done = torch.cuda.Event()
                done.record(main)
                side.wait_event(done)
            if timer is not None:
                timer.start("peaks", side)
            R.retina_find_peaks(out, sp.P, sp.peak_threshold, sp.peak_capacity,
                                out=(self.peak_idx[e0:e1], self.peak_val[e0:e1], self.peak_cnt[e0:e1]),
                                stream=side, workspace=self.peak_ws)
            # step (iv): sub-cell parameter estimate of every peak
            R.retina_estimate_peaks(out, self.nodes, self.peak_idx[e0:e1], self.peak_cnt[e0:e1],
                                    out=self.peak_theta[e0:e1], stream=side)
            if timer is not None:
                timer.stop("peaks", side)
            if side is not main:
                freed[b] = torch.cuda.Event()
                freed[b].record(side)
            self.launches += 3 + (1 if self.peak_ws is not None else 0)  # slab peaks = 2 kernels
        if side is not main:
            main.wait_stream(side)

    def run_multistart(self, batch: DeviceBatch, stream=None, timer=None):
        sp = self.spec
        E = batch.n_events
        ev = self.events_view(batch, 0, E)
        if timer is not None:
            timer.start("multistart")
        if sp.newton is not None:  # the paper's update: Truncated Newton with a sigma schedule
            sig, eta, fsig, mh = sp.newton
            R.retina_multistart_newton_ex(ev, sp.model, batch.seeds, sig, eta, fsig, mh, sp.box_lo, sp.box_hi,
                                          want_grad=False, out=(self.theta[:E], self.resp[:E], None, self.evals[:E]),
                                          stream=stream, algorithm=sp.ms_algorithm, workspace=self.ms_ws,
                                          pairs_evaluated=self.pairs_ev if self.count_pairs else None)
        else:  # BASELINE configs[2..4]: fixed-step gradient ascent
            R.retina_multistart_optimize(ev, sp.model, sp.sigma_ms or sp.sigma, batch.seeds, sp.n_iters, sp.step,
                                         sp.box_lo, sp.box_hi, want_grad=False,
                                         out=(self.theta[:E], self.resp[:E], None), stream=stream,
                                         algorithm=sp.ms_algorithm, workspace=self.ms_ws,
                                         pairs_evaluated=self.pairs_ev if self.count_pairs else None)
        if timer is not None:
            timer.stop("multistart")
            timer.start("merge")
        R.retina_merge_tracks(self.theta[:E], self.resp[:E], sp.merge_radius, sp.track_threshold,
                              sp.track_capacity,
                              out=(self.t_theta[:E], self.t_resp[:E], self.t_seed[:E], self.t_size[:E],
                                   self.t_count[:E]), stream=stream)
        if timer is not None:
            timer.stop("merge")
        self.launches += 2

    def run(self, batch: DeviceBatch, stream=None, timer=None):
        if self.spec.cells:
            self.run_grid(batch, stream, timer)
        if self.spec.n_seeds:
            self.run_multistart(batch, stream, timer)

    def capture(self, batch: DeviceBatch) -> "torch.cuda.CUDAGraph":
        """Records one whole pass (every kernel launch of run()) into a CUDA graph; replaying it
        re-runs the hot path on whatever is in `batch`'s device buffers, with no host work per
        launch.  The library keeps no launch-time state besides its smem-attribute cache, which
        the eager warm-up pass fills, so capture contains kernel launches only."""
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.run(batch)  # warm-up outside capture (attribute cache, lazy module loading)
        torch.cuda.current_stream(self.device).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.run(batch)
        return graph


class PhaseTimer:
    """CUDA-event timer per phase on a given stream: per step, the sum over the phase's launches;
    reported as the median over steps (median of >= 5 timed repetitions)."""

    def __init__(self, stream):
        self.stream = stream
        self.pending = {}
        self.events: dict = {}
        self.cur = 0

    def next_step(self):
        self.cur += 1

    def start(self, name, stream=None):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream or self.stream)
        self.pending[name] = ev

    def stop(self, name, stream=None):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream or self.stream)
        self.events.setdefault(name, []).append((self.pending.pop(name), ev, self.cur))

    def per_step_ms(self):
        """{phase: [ms of step 0, step 1, ...]} (sum over the phase's launches in each step)."""
        out = {}
        for k, v in self.events.items():
            steps = {}
            for a, b, st in v:
                steps[st] = steps.get(st, 0.0) + a.elapsed_time(b)
            out[k] = [steps[st] for st in sorted(steps)]
        return out

    def totals_ms(self):
        return {k: sum(v) for k, v in self.per_step_ms().items()}

    def counts(self):
        return {k: len(v) for k, v in self.events.items()}

    def reset(self):
        self.events = {}
        self.pending = {}
        self.cur = 0


def upload(offsets: np.ndarray, hits: np.ndarray, seeds: np.ndarray, device="cuda",
           pinned: bool = False, stream=None) -> DeviceBatch:
    """Host -> device copy of one batch (from pinned buffers when `pinned`)."""
    def t(a, dtype):
        x = torch.from_numpy(np.ascontiguousarray(a))
        if pinned:
            x = x.pin_memory()
        return x.to(device, dtype, non_blocking=pinned)
    counts = np.diff(np.asarray(offsets, np.int64))
    return DeviceBatch(offsets=t(offsets.astype(np.int32), torch.int32), hits=t(hits, torch.float32),
                       seeds=t(seeds, torch.float32),
                       max_event_hits=int(counts.max()) if len(counts) else 0, n_hits_per_event=counts)
