"""Event-parallel multi-GPU plumbing.

Events are independent ("extremely high parallelization capacity"; north star
"Events are independent"), so rank r of W owns the contiguous block
[floor(r E / W), floor((r + 1) E / W)) of the batch and runs the whole hot path on its own GPU
with no data-path collective.  The only exchange is ONE all_gather_into_tensor of a fixed-size
per-rank record (found peaks and tracks, first `keep` per event, plus a header with the rank's
event range, totals and work) -- "one NCCL gather over NVLink for found tracks and timings
only".  The record is written on the device by libretina's retina_pack_results kernel;
torch.distributed only moves it.  The per-rank step timings are gathered once, after the
timed region (bench.py).
"""
from __future__ import annotations

import os
import struct
from typing import Dict, List, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import retina as RT

HEADER = RT.PACK_HEADER  # words: rank, event_base, n_events, peaks_total, tracks_total, pairs_grid/1e9, pairs_ms/1e9, 0


def env() -> Tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [floor(r E / W), floor((r+1) E / W)) of a fixed event set."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def record_width(P: int, keep: int) -> int:
    """32-bit words per event (RETINA_PACK_WORDS)."""
    return RT.pack_words(P, keep)


def _f32_bits(v: float) -> int:
    return struct.unpack("<I", struct.pack("<f", float(v)))[0]


def header_words(rank: int, event_base: int, n_events: int, pairs_grid: float, pairs_ms: float) -> List[int]:
    """The host part of the record header (the totals, words 3 and 4, are summed on the device)."""
    return [rank, event_base, n_events, 0, 0, _f32_bits(pairs_grid / 1e9), _f32_bits(pairs_ms / 1e9), 0]


def pack(peak_idx, peak_val, peak_cnt, t_theta, t_resp, t_size, t_count, keep: int, header: List[int],
         out=None, stream=None) -> torch.Tensor:
    """The rank's record, written on the device by retina_pack_results (int32 words)."""
    return RT.retina_pack_results(peak_idx, peak_val, peak_cnt, t_theta, t_resp, t_size, t_count, keep, header,
                                  out=out, stream=stream)


def gather(buf: torch.Tensor, world: int) -> torch.Tensor:
    """THE one collective: all_gather_into_tensor of equal-size per-rank buffers."""
    if world == 1:
        return buf[None]
    out = torch.empty((world, buf.numel()), dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(out.view(-1), buf)
    return out


def unpack(gathered: np.ndarray, P: int, keep: int) -> List[Dict]:
    """Host-side decode of the gathered records (rank order)."""
    out = []
    w = record_width(P, keep)
    g = np.ascontiguousarray(np.asarray(gathered)).astype(np.int32, copy=False)
    for row in g:
        hdr = row[:HEADER]
        hf = hdr.view(np.float32)
        E = int(hdr[2])
        rec = row[HEADER:HEADER + E * w].reshape(E, w)
        recf = rec.view(np.float32)
        o = 2 + 2 * keep
        tr = recf[:, o:].reshape(E, keep, P + 2).astype(np.float64)
        tr[:, :, P + 1] = rec[:, o:].reshape(E, keep, P + 2)[:, :, P + 1]  # size is an integer word
        out.append(dict(rank=int(hdr[0]), event_base=int(hdr[1]), n_events=E,
                        peaks_total=int(np.uint32(hdr[3])), tracks_total=int(np.uint32(hdr[4])),
                        pairs_grid=float(hf[5]) * 1e9, pairs_ms=float(hf[6]) * 1e9,
                        n_peaks=rec[:, 0].astype(np.int64), n_tracks=rec[:, 1].astype(np.int64),
                        peak_index=rec[:, 2:2 + keep].astype(np.int64),
                        peak_value=recf[:, 2 + keep:2 + 2 * keep].astype(np.float64),
                        tracks=tr))
    return out
