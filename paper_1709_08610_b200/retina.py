"""Thin Python binding of libretina.so (include/retina.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind
the C ABI.  torch is used for device memory and streams.  There is no CPU fallback: if
the shared library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

from .build import LIB

LINE2D, SLOPE2, SLOPE3 = 0, 1, 2
MODEL_P = {LINE2D: 2, SLOPE2: 2, SLOPE3: 3}
RETINA_OK, RETINA_EINVAL, RETINA_EUNSUPPORTED, RETINA_ECUDA = 0, 1, 2, 3
MERGE_MAX_SEEDS = 16384

GRID_AUTO, GRID_DIRECT, GRID_SEPARABLE, GRID_TENSOR, GRID_TENSOR_F16 = 0, 1, 2, 3, 4
GRID_TENSOR_F16_PAIR, GRID_TENSOR_F16_SINGLE, GRID_TENSOR_F16_CULLED = 5, 6, 7
MS_DENSE, MS_CULLED = 0, 1

EXPORTED = ("retina_grid_response", "retina_grid_response_ex", "retina_grid_response_ex2", "retina_estimate_peaks",
            "retina_find_peaks",
            "retina_find_peaks_ws", "retina_find_peaks_workspace_size",
            "retina_multistart_optimize", "retina_multistart_optimize_ex", "retina_multistart_workspace_size",
            "retina_multistart_newton", "retina_multistart_newton_ex", "retina_multistart_newton_ex2",
            "retina_merge_tracks", "retina_pack_results",
            "retina_status_string", "retina_last_error", "retina_version")
PACK_HEADER = 8


def pack_words(P: int, keep: int) -> int:
    """RETINA_PACK_WORDS(P, keep): 32-bit words per event in a retina_pack_results record."""
    return 2 + 2 * keep + keep * (P + 2)


class RetinaError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str):
        super().__init__(f"{fn} -> {status}: {detail}")
        self.status = status


class retina_events(ctypes.Structure):
    _fields_ = [("n_events", ctypes.c_int32), ("offsets", ctypes.c_void_p), ("hits", ctypes.c_void_p),
                ("z_ref", ctypes.c_float), ("max_event_hits", ctypes.c_int32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libretina.so (built in-tree by __graft_entry__.build() / build.py)."""
    global _lib
    if _lib is None:
        path = os.environ.get("RETINA_LIB", LIB)  # experiments may point at a variant build
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_1709_08610_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        vp, i32, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float
        L.retina_grid_response.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, f32, vp, vp, vp, vp]
        L.retina_grid_response_ex2.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, f32, vp, vp, vp,
                                               ctypes.c_int, vp, vp]
        L.retina_grid_response_ex2.restype = ctypes.c_int
        L.retina_grid_response_ex.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, f32, vp, vp, vp,
                                              ctypes.c_int, vp]
        L.retina_find_peaks.argtypes = [vp, i32, i32, vp, f32, i32, vp, vp, vp, vp]
        L.retina_estimate_peaks.argtypes = [vp, i32, i32, vp, vp, vp, vp, i32, vp, vp]
        L.retina_find_peaks_ws.argtypes = [vp, i32, i32, vp, f32, i32, vp, vp, vp, vp, ctypes.c_size_t, vp]
        L.retina_find_peaks_ws.restype = ctypes.c_int
        L.retina_find_peaks_workspace_size.argtypes = [i32, i32, vp]
        L.retina_find_peaks_workspace_size.restype = ctypes.c_size_t
        L.retina_multistart_optimize.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, f32, i32, vp,
                                                 i32, f32, vp, vp, vp, vp, vp, vp]
        L.retina_multistart_optimize_ex.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, f32, i32, vp,
                                                    i32, f32, vp, vp, vp, vp, vp, ctypes.c_int, vp,
                                                    ctypes.c_size_t, vp, vp]
        L.retina_multistart_workspace_size.argtypes = [i32, i32, ctypes.c_int]
        L.retina_multistart_workspace_size.restype = ctypes.c_size_t
        L.retina_multistart_newton.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, i32, vp, i32, vp, vp,
                                               f32, i32, vp, vp, vp, vp, vp, vp]
        L.retina_multistart_newton_ex.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, i32, vp, i32, vp,
                                                  vp, f32, i32, vp, vp, vp, vp, vp, vp, vp]
        L.retina_multistart_newton_ex2.argtypes = [ctypes.POINTER(retina_events), ctypes.c_int, i32, vp, i32, vp,
                                                   vp, f32, i32, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp,
                                                   ctypes.c_size_t, vp, vp]
        L.retina_merge_tracks.argtypes = [i32, i32, i32, vp, vp, vp, f32, i32, vp, vp, vp, vp, vp, vp]
        L.retina_pack_results.argtypes = [i32, i32, i32, vp, vp, vp, i32, vp, vp, vp, vp, i32, vp, vp, vp]
        for f in (L.retina_grid_response, L.retina_grid_response_ex, L.retina_find_peaks, L.retina_estimate_peaks,
                  L.retina_multistart_optimize, L.retina_multistart_optimize_ex, L.retina_multistart_newton,
                  L.retina_multistart_newton_ex, L.retina_multistart_newton_ex2,
                  L.retina_merge_tracks, L.retina_pack_results):
            f.restype = ctypes.c_int
        L.retina_status_string.argtypes = [ctypes.c_int]
        L.retina_status_string.restype = ctypes.c_char_p
        L.retina_last_error.restype = ctypes.c_char_p
        L.retina_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def version() -> str:
    return lib().retina_version().decode()


def _check(fn: str, status: int):
    if status != RETINA_OK:
        raise RetinaError(fn, status, lib().retina_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _arr(ctype, vals):
    a = (ctype * max(len(vals), 1))(*vals)
    return ctypes.cast(a, ctypes.c_void_p), a  # keep `a` alive while the call runs


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, dtype) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError("device tensor expected (the library takes device pointers)")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"contiguous {dtype} tensor expected")
    return t


def _out(name: str, t: Optional[torch.Tensor], dtype, shape, device) -> Optional[torch.Tensor]:
    """Checks a caller-supplied output buffer before its raw pointer reaches a kernel: CUDA,
    contiguous, the expected dtype, shape and device (a narrower buffer would be written out
    of bounds, not rejected, by the device code)."""
    if t is None:
        return None
    _dev(t, dtype)
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)} expected {tuple(shape)}")
    if t.device != device:
        raise ValueError(f"{name}: on {t.device}, inputs on {device}")
    return t


class Events:
    """A device-resident CSR batch: offsets int32 [E+1], hits float32 [N, 4]."""

    def __init__(self, offsets: torch.Tensor, hits: torch.Tensor, z_ref: float = 0.0,
                 max_event_hits: int = 0):
        self.offsets = _dev(offsets, torch.int32)
        self.hits = _dev(hits, torch.float32)
        assert hits.dim() == 2 and hits.shape[1] == 4
        self.n_events = offsets.numel() - 1
        self.c = retina_events(self.n_events, offsets.data_ptr(), hits.data_ptr(), float(z_ref),
                               int(max_event_hits))

    @staticmethod
    def from_numpy(offsets, hits, z_ref: float = 0.0, device="cuda", max_event_hits: Optional[int] = None):
        import numpy as np
        off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int32)).to(device)
        h = torch.from_numpy(np.ascontiguousarray(hits, dtype=np.float32)).to(device)
        if max_event_hits is None:
            o = np.asarray(offsets)
            max_event_hits = int(np.max(np.diff(o))) if len(o) > 1 else 0
        return Events(off, h, z_ref, max_event_hits)


def grid_shape(n_events: int, axis_len: Sequence[int]) -> tuple:
    """Shape of a response grid: (E, n0, n1) for P = 2, (E, n2, n0, n1) for P = 3 -- one (tx, ty)
    plane per z0 node (retina.h; Z37)."""
    n = [int(v) for v in axis_len]
    return (int(n_events),) + ((n[2], n[0], n[1]) if len(n) == 3 else tuple(n))


def _param_axis_len(grid_dims: Sequence[int]) -> list:
    """Per-event grid dims (memory order) -> axis_len in parameter order (tx, ty[, z0])."""
    d = [int(v) for v in grid_dims]
    return [d[1], d[2], d[0]] if len(d) == 3 else d


def retina_grid_response(events: Events, model: int, sigma: float, nodes: Sequence[torch.Tensor],
                         out: Optional[torch.Tensor] = None, stream=None, algorithm: int = GRID_AUTO,
                         pairs_evaluated: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Eq. (2) grid, shape grid_shape(E, node counts).  pairs_evaluated (int64 [1] device tensor)
    accumulates the (unit, hit) pairs contracted (retina_grid_response_ex2)."""
    P = MODEL_P[model]
    nodes = [_dev(n, torch.float32) for n in nodes]
    alen, _k1 = _arr(ctypes.c_int32, [n.numel() for n in nodes])
    nptr, _k2 = _arr(ctypes.c_void_p, [n.data_ptr() for n in nodes])
    shape = grid_shape(events.n_events, [n.numel() for n in nodes])
    if out is None:
        out = torch.empty(shape, device=events.hits.device, dtype=torch.float32)
    _out("response", out, torch.float32, shape, events.hits.device)
    if pairs_evaluated is not None:
        _out("pairs_evaluated", pairs_evaluated, torch.int64, (1,), events.hits.device)
        _check("retina_grid_response_ex2",
               lib().retina_grid_response_ex2(ctypes.byref(events.c), model, float(sigma), alen, nptr,
                                              _ptr(_dev(out, torch.float32)), int(algorithm), _ptr(pairs_evaluated),
                                              _stream(stream)))
        return out
    _check("retina_grid_response_ex",
           lib().retina_grid_response_ex(ctypes.byref(events.c), model, float(sigma), alen, nptr,
                                         _ptr(_dev(out, torch.float32)), int(algorithm), _stream(stream)))
    return out


def find_peaks_workspace_size(n_events: int, shape) -> int:
    """Workspace bytes of retina_find_peaks_ws for grids of per-event shape `shape` (the response
    tensor's shape[1:], memory order)."""
    alen, _k = _arr(ctypes.c_int32, _param_axis_len(shape))
    return int(lib().retina_find_peaks_workspace_size(int(n_events), len(shape), alen))


def retina_find_peaks(response: torch.Tensor, P: int, threshold: float, capacity: int,
                      out=None, stream=None, workspace: Optional[torch.Tensor] = None):
    """Returns (peak_index int32 [E, cap], peak_value fp32 [E, cap], peak_count int32 [E]).
    With a device `workspace` (>= find_peaks_workspace_size bytes) the many-CTA path
    (retina_find_peaks_ws) is used; the results are identical."""
    _dev(response, torch.float32)
    E = response.shape[0]
    shape = tuple(response.shape[1:])
    assert len(shape) == P
    alen, _k = _arr(ctypes.c_int32, _param_axis_len(shape))
    if out is None:
        dev = response.device
        out = (torch.empty((E, capacity), dtype=torch.int32, device=dev),
               torch.empty((E, capacity), dtype=torch.float32, device=dev),
               torch.empty((E,), dtype=torch.int32, device=dev))
    idx, val, cnt = out
    _out("peak_index", idx, torch.int32, (E, capacity), response.device)
    _out("peak_value", val, torch.float32, (E, capacity), response.device)
    _out("peak_count", cnt, torch.int32, (E,), response.device)
    if workspace is not None:
        _dev(workspace, workspace.dtype)
        if workspace.device != response.device:
            raise ValueError("workspace on another device")
        nbytes = workspace.numel() * workspace.element_size()
        _check("retina_find_peaks_ws",
               lib().retina_find_peaks_ws(_ptr(response), E, P, alen, float(threshold), int(capacity), _ptr(idx),
                                          _ptr(val), _ptr(cnt), _ptr(workspace), ctypes.c_size_t(nbytes),
                                          _stream(stream)))
    else:
        _check("retina_find_peaks",
               lib().retina_find_peaks(_ptr(response), E, P, alen, float(threshold), int(capacity),
                                       _ptr(idx), _ptr(val), _ptr(cnt), _stream(stream)))
    return idx, val, cnt


def retina_estimate_peaks(response: torch.Tensor, nodes: Sequence[torch.Tensor], peak_index: torch.Tensor,
                          peak_count: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Step (iv): per-peak quadratic sub-cell estimate, fp32 [E, capacity, P]."""
    _dev(response, torch.float32)
    nodes = [_dev(n, torch.float32) for n in nodes]
    P = len(nodes)
    E, cap = peak_index.shape
    alen, _k1 = _arr(ctypes.c_int32, [n.numel() for n in nodes])
    nptr, _k2 = _arr(ctypes.c_void_p, [n.data_ptr() for n in nodes])
    if tuple(response.shape) != grid_shape(E, [n.numel() for n in nodes]):
        raise ValueError("response must be grid_shape(E, node counts) with E = peak_index.shape[0]")
    _out("peak_count", _dev(peak_count, torch.int32), torch.int32, (E,), response.device)
    if out is None:
        out = torch.zeros((E, cap, P), dtype=torch.float32, device=response.device)
    _out("theta", out, torch.float32, (E, cap, P), response.device)
    _check("retina_estimate_peaks",
           lib().retina_estimate_peaks(_ptr(response), E, P, alen, nptr, _ptr(_dev(peak_index, torch.int32)),
                                       _ptr(_dev(peak_count, torch.int32)), int(cap), _ptr(out), _stream(stream)))
    return out


def retina_multistart_optimize(events: Events, model: int, sigma: float, seeds: torch.Tensor,
                               n_iters: int, step: float, box_lo, box_hi, want_grad: bool = True,
                               out=None, stream=None, algorithm: int = MS_DENSE,
                               workspace: Optional[torch.Tensor] = None,
                               pairs_evaluated: Optional[torch.Tensor] = None):
    """Returns (theta_out [E,S,P], response_out [E,S], grad_out [E,S,P] or None).  algorithm=MS_CULLED
    (SLOPE2) gives the same results bit for bit evaluating only the pairs that can contribute
    (retina_multistart_optimize_ex; a workspace is allocated if none is passed); pairs_evaluated, an
    int64 [1] device tensor, accumulates the pairs actually evaluated."""
    P = MODEL_P[model]
    _dev(seeds, torch.float32)
    E, S, Ps = seeds.shape
    assert Ps == P and E == events.n_events
    lo, _k1 = _arr(ctypes.c_float, [float(v) for v in box_lo])
    hi, _k2 = _arr(ctypes.c_float, [float(v) for v in box_hi])
    if out is None:
        out = (torch.empty_like(seeds), torch.empty((E, S), dtype=torch.float32, device=seeds.device),
               torch.empty_like(seeds) if want_grad else None)
    th, R, g = out
    _out("theta_out", th, torch.float32, (E, S, P), seeds.device)
    _out("response_out", R, torch.float32, (E, S), seeds.device)
    _out("grad_out", g, torch.float32, (E, S, P), seeds.device)
    if algorithm == MS_DENSE and workspace is None and pairs_evaluated is None:
        _check("retina_multistart_optimize",
               lib().retina_multistart_optimize(ctypes.byref(events.c), model, float(sigma), S, _ptr(seeds),
                                                int(n_iters), float(step), lo, hi, _ptr(th), _ptr(R), _ptr(g),
                                                _stream(stream)))
        return th, R, g
    if algorithm == MS_CULLED and workspace is None:
        nbytes = multistart_workspace_size(E, S, algorithm)
        workspace = torch.empty((max(nbytes, 4) // 4,), dtype=torch.int32, device=seeds.device)
    nbytes = 0
    if workspace is not None:
        _dev(workspace, workspace.dtype)
        if workspace.device != seeds.device:
            raise ValueError("workspace on another device")
        nbytes = workspace.numel() * workspace.element_size()
    if pairs_evaluated is not None:
        _out("pairs_evaluated", pairs_evaluated, torch.int64, (1,), seeds.device)
    _check("retina_multistart_optimize_ex",
           lib().retina_multistart_optimize_ex(ctypes.byref(events.c), model, float(sigma), S, _ptr(seeds),
                                               int(n_iters), float(step), lo, hi, _ptr(th), _ptr(R), _ptr(g),
                                               int(algorithm), _ptr(workspace), ctypes.c_size_t(nbytes),
                                               _ptr(pairs_evaluated), _stream(stream)))
    return th, R, g


def multistart_workspace_size(n_events: int, n_seeds: int, algorithm: int = MS_CULLED) -> int:
    """Bytes of device workspace retina_multistart_optimize_ex and retina_multistart_newton_ex2 need
    (0 for MS_DENSE)."""
    return int(lib().retina_multistart_workspace_size(int(n_events), int(n_seeds), int(algorithm)))


def retina_multistart_newton(events: Events, model: int, seeds: torch.Tensor, sigmas, etas, final_sigma: float,
                             max_halvings: int, box_lo, box_hi, want_grad: bool = True, out=None, stream=None):
    """Truncated-Newton multi-start: (theta_out, response_out, grad_out or None)."""
    return _newton(False, events, model, seeds, sigmas, etas, final_sigma, max_halvings, box_lo, box_hi, want_grad,
                   out, stream)[:3]


def retina_multistart_newton_ex(events: Events, model: int, seeds: torch.Tensor, sigmas, etas, final_sigma: float,
                                max_halvings: int, box_lo, box_hi, want_grad: bool = True, out=None, stream=None,
                                algorithm: int = MS_DENSE, workspace: Optional[torch.Tensor] = None,
                                pairs_evaluated: Optional[torch.Tensor] = None):
    """As retina_multistart_newton, plus the per-seed response-evaluation counts (int32 [E, S]):
    (theta_out, response_out, grad_out or None, evals_out).  algorithm=MS_CULLED (or a
    pairs_evaluated int64 [1] device tensor) goes through retina_multistart_newton_ex2: the same
    results bit for bit, each warp visiting only the hits that can contribute (a workspace is
    allocated if none is passed)."""
    return _newton(True, events, model, seeds, sigmas, etas, final_sigma, max_halvings, box_lo, box_hi, want_grad,
                   out, stream, algorithm, workspace, pairs_evaluated)


def _newton(ex, events, model, seeds, sigmas, etas, final_sigma, max_halvings, box_lo, box_hi, want_grad, out,
            stream, algorithm=MS_DENSE, workspace=None, pairs_evaluated=None):
    P = MODEL_P[model]
    _dev(seeds, torch.float32)
    E, S, Ps = seeds.shape
    assert Ps == P and E == events.n_events and len(sigmas) == len(etas)
    sg, _k1 = _arr(ctypes.c_float, [float(v) for v in sigmas])
    et, _k2 = _arr(ctypes.c_float, [float(v) for v in etas])
    lo, _k3 = _arr(ctypes.c_float, [float(v) for v in box_lo])
    hi, _k4 = _arr(ctypes.c_float, [float(v) for v in box_hi])
    if out is None:
        out = (torch.empty_like(seeds), torch.empty((E, S), dtype=torch.float32, device=seeds.device),
               torch.empty_like(seeds) if want_grad else None)
        if ex:
            out = out + (torch.empty((E, S), dtype=torch.int32, device=seeds.device),)
    th, R, g = out[:3]
    _out("theta_out", th, torch.float32, (E, S, P), seeds.device)
    _out("response_out", R, torch.float32, (E, S), seeds.device)
    _out("grad_out", g, torch.float32, (E, S, P), seeds.device)
    if ex:
        ne = out[3] if len(out) > 3 and out[3] is not None else torch.empty((E, S), dtype=torch.int32,
                                                                           device=seeds.device)
        _out("evals_out", ne, torch.int32, (E, S), seeds.device)
        if algorithm != MS_DENSE or workspace is not None or pairs_evaluated is not None:
            if algorithm == MS_CULLED and workspace is None:
                nbytes = multistart_workspace_size(E, S, algorithm)
                workspace = torch.empty((max(nbytes, 4) // 4,), dtype=torch.int32, device=seeds.device)
            nbytes = 0
            if workspace is not None:
                _dev(workspace, workspace.dtype)
                if workspace.device != seeds.device:
                    raise ValueError("workspace on another device")
                nbytes = workspace.numel() * workspace.element_size()
            if pairs_evaluated is not None:
                _out("pairs_evaluated", pairs_evaluated, torch.int64, (1,), seeds.device)
            _check("retina_multistart_newton_ex2",
                   lib().retina_multistart_newton_ex2(ctypes.byref(events.c), model, S, _ptr(seeds), len(sigmas), sg,
                                                      et, float(final_sigma), int(max_halvings), lo, hi, _ptr(th),
                                                      _ptr(R), _ptr(g), _ptr(ne), int(algorithm), _ptr(workspace),
                                                      ctypes.c_size_t(nbytes), _ptr(pairs_evaluated), _stream(stream)))
            return th, R, g, ne
        _check("retina_multistart_newton_ex",
               lib().retina_multistart_newton_ex(ctypes.byref(events.c), model, S, _ptr(seeds), len(sigmas), sg, et,
                                                 float(final_sigma), int(max_halvings), lo, hi, _ptr(th), _ptr(R),
                                                 _ptr(g), _ptr(ne), _stream(stream)))
        return th, R, g, ne
    _check("retina_multistart_newton",
           lib().retina_multistart_newton(ctypes.byref(events.c), model, S, _ptr(seeds), len(sigmas), sg, et,
                                          float(final_sigma), int(max_halvings), lo, hi, _ptr(th), _ptr(R),
                                          _ptr(g), _stream(stream)))
    return th, R, g


def retina_merge_tracks(theta: torch.Tensor, response: torch.Tensor, radius, threshold: float,
                        capacity: int, out=None, stream=None):
    """Returns (track_theta [E,cap,P], track_response [E,cap], track_seed, track_size, track_count)."""
    _dev(theta, torch.float32)
    _dev(response, torch.float32)
    E, S, P = theta.shape
    rad, _k = _arr(ctypes.c_float, [float(v) for v in radius])
    if out is None:
        dev = theta.device
        out = (torch.empty((E, capacity, P), dtype=torch.float32, device=dev),
               torch.empty((E, capacity), dtype=torch.float32, device=dev),
               torch.empty((E, capacity), dtype=torch.int32, device=dev),
               torch.empty((E, capacity), dtype=torch.int32, device=dev),
               torch.empty((E,), dtype=torch.int32, device=dev))
    tt, tr, ts, tz, tc = out
    for nm, t, dt, shp in (("track_theta", tt, torch.float32, (E, capacity, P)),
                           ("track_response", tr, torch.float32, (E, capacity)),
                           ("track_seed", ts, torch.int32, (E, capacity)), ("track_size", tz, torch.int32, (E, capacity)),
                           ("track_count", tc, torch.int32, (E,))):
        _out(nm, t, dt, shp, theta.device)
    _check("retina_merge_tracks",
           lib().retina_merge_tracks(E, S, P, _ptr(theta), _ptr(response), rad, float(threshold), int(capacity),
                                     _ptr(tt), _ptr(tr), _ptr(ts), _ptr(tz), _ptr(tc), _stream(stream)))
    return tt, tr, ts, tz, tc


def retina_pack_results(peak_index: torch.Tensor, peak_value: torch.Tensor, peak_count: torch.Tensor,
                        track_theta: torch.Tensor, track_response: torch.Tensor, track_size: torch.Tensor,
                        track_count: torch.Tensor, keep: int, header, out: Optional[torch.Tensor] = None,
                        stream=None) -> torch.Tensor:
    """The per-rank record of the one result gather: int32 [PACK_HEADER + E * pack_words(P, keep)]
    (fp32 fields as bit patterns).  `header`: PACK_HEADER uint32 words (see dist.header_words)."""
    E, pcap = peak_index.shape
    _, tcap, P = track_theta.shape
    dev = peak_index.device
    _out("peak_index", peak_index, torch.int32, (E, pcap), dev)
    _out("peak_value", peak_value, torch.float32, (E, pcap), dev)
    _out("peak_count", peak_count, torch.int32, (E,), dev)
    _out("track_theta", track_theta, torch.float32, (E, tcap, P), dev)
    _out("track_response", track_response, torch.float32, (E, tcap), dev)
    _out("track_size", track_size, torch.int32, (E, tcap), dev)
    _out("track_count", track_count, torch.int32, (E,), dev)
    n = PACK_HEADER + E * pack_words(P, keep)
    if out is None:
        out = torch.empty((n,), dtype=torch.int32, device=dev)
    _out("out", out, torch.int32, (n,), dev)
    hdr = list(header)
    if len(hdr) != PACK_HEADER:
        raise ValueError(f"header needs {PACK_HEADER} words")
    h, _k = _arr(ctypes.c_uint32, [int(v) & 0xFFFFFFFF for v in hdr])
    _check("retina_pack_results",
           lib().retina_pack_results(E, P, int(keep), _ptr(peak_index), _ptr(peak_value), _ptr(peak_count), pcap,
                                     _ptr(track_theta), _ptr(track_response), _ptr(track_size), _ptr(track_count),
                                     tcap, h, _ptr(out), _stream(stream)))
    return out
