"""Event-parallel multi-GPU plumbing.

Events are independent ("extremely high parallelization capacity"; north star
"Events are independent"), so rank r of W owns a contiguous block of event ids and runs the
whole hot path on its own GPU with no data-path collective.  The only exchange is ONE
all_gather_into_tensor of a fixed-size per-rank record buffer holding the found peaks and
tracks (first `keep` per event) and the rank's timings -- "one NCCL gather over NVLink for
found tracks and timings only".  The same code runs on gloo over CPU tensors in the tests.
"""
from __future__ import annotations

import os
from typing import Dict, List, Tuple

import numpy as np
import torch
import torch.distributed as dist

HEADER = 8  # floats: rank, event_base, n_events, peaks_total, tracks_total, t_ms, pairs_grid/1e9, pairs_ms/1e9


def env() -> Tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [floor(r E / W), floor((r+1) E / W)) of a fixed event set."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def record_width(P: int, keep: int) -> int:
    # per event: n_peaks, n_tracks, keep x (peak index, peak value), keep x (theta[P], R, size)
    return 2 + 2 * keep + keep * (P + 2)


def pack(peak_idx, peak_val, peak_cnt, t_theta, t_resp, t_size, t_count, keep: int,
         header: List[float]) -> torch.Tensor:
    """Fixed-size float32 buffer [HEADER + E * record_width] (device tensor ops only)."""
    E = peak_cnt.shape[0]
    P = t_theta.shape[2]
    k1 = min(keep, peak_idx.shape[1])
    k2 = min(keep, t_theta.shape[1])
    dev = peak_cnt.device
    rec = torch.zeros((E, record_width(P, keep)), dtype=torch.float32, device=dev)
    rec[:, 0] = peak_cnt.float()
    rec[:, 1] = t_count.float()
    rec[:, 2:2 + keep] = -1.0
    o = 2
    pk = torch.arange(k1, device=dev)[None, :] < peak_cnt[:, None]
    rec[:, o:o + k1] = torch.where(pk, peak_idx[:, :k1].float(), torch.full_like(peak_val[:, :k1], -1))
    rec[:, o + keep:o + keep + k1] = torch.where(pk, peak_val[:, :k1], torch.zeros_like(peak_val[:, :k1]))
    o += 2 * keep
    tk = (torch.arange(k2, device=dev)[None, :] < t_count[:, None]).float()
    tr = torch.cat([t_theta[:, :k2], t_resp[:, :k2, None], t_size[:, :k2, None].float()], dim=2)
    tr = tr * tk[:, :, None]
    rec[:, o:o + k2 * (P + 2)] = tr.reshape(E, -1)
    # header: host-known values, with the two totals summed on the device (no host sync)
    hdr = torch.tensor(header, dtype=torch.float32, device=dev)
    hdr[3] = peak_cnt.sum().float()
    hdr[4] = t_count.sum().float()
    return torch.cat([hdr, rec.reshape(-1)])


def gather(buf: torch.Tensor, world: int) -> torch.Tensor:
    """THE one collective: all_gather_into_tensor of equal-size per-rank buffers."""
    if world == 1:
        return buf[None]
    out = torch.empty((world, buf.numel()), dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(out.view(-1), buf)
    return out


def unpack(gathered: np.ndarray, P: int, keep: int) -> List[Dict]:
    """Host-side decode of the gathered buffers (rank order)."""
    out = []
    w = record_width(P, keep)
    for row in np.asarray(gathered, np.float64):
        hdr = row[:HEADER]
        E = int(hdr[2])
        rec = row[HEADER:HEADER + E * w].reshape(E, w)
        o = 2 + 2 * keep
        tracks = rec[:, o:].reshape(E, keep, P + 2)
        out.append(dict(rank=int(hdr[0]), event_base=int(hdr[1]), n_events=E,
                        peaks_total=int(hdr[3]), tracks_total=int(hdr[4]), t_ms=float(hdr[5]),
                        pairs_grid=hdr[6] * 1e9, pairs_ms=hdr[7] * 1e9,
                        n_peaks=rec[:, 0].astype(np.int64), n_tracks=rec[:, 1].astype(np.int64),
                        peak_index=rec[:, 2:2 + keep].astype(np.int64), peak_value=rec[:, 2 + keep:2 + 2 * keep],
                        tracks=tracks))
    return out
