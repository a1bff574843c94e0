"""N>1 host logic on CPU: sharding, the pack -> all_gather_into_tensor -> unpack round trip
over gloo with world_size 2, and world-size invariance of the keyed inputs."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1709_08610_b200 import dist as D
from synth import configs as C
from synth import events as G
from tests.pack_ref import pack_ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_exactly():
    for n in (0, 1, 7, 10000):
        for w in (1, 2, 3, 8):
            blocks = [D.shard(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))


def _fake_results(rank, E, P, cap, seed):
    g = torch.Generator().manual_seed(seed + rank)
    pc = torch.randint(0, cap + 3, (E,), generator=g, dtype=torch.int32)
    pi = torch.randint(0, 1000, (E, cap), generator=g, dtype=torch.int32)
    pv = torch.rand((E, cap), generator=g)
    tc = torch.randint(0, cap + 3, (E,), generator=g, dtype=torch.int32)
    tt = torch.rand((E, cap, P), generator=g)
    tr = torch.rand((E, cap), generator=g) * 10
    tz = torch.randint(1, 9, (E, cap), generator=g, dtype=torch.int32)
    return pi, pv, pc, tt, tr, tz, tc


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    E, P, cap, keep = 5, 3, 6, 4
    res = _fake_results(rank, E, P, cap, 0)
    # the record as retina_pack_results lays it out (the device kernel is checked against the same
    # reference word for word in tests/test_parity_gpu.py); here gloo moves it
    buf = torch.from_numpy(pack_ref(*(x.numpy() for x in res), keep,
                                    D.header_words(rank, rank * E, E, 1.5e9 * (rank + 1), 2.5e9)))
    gathered = D.gather(buf, world)
    if rank == 0:
        np.save(out_path, gathered.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_pack_gather_unpack_gloo_world2(tmp_path):
    out = str(tmp_path / "g.npy")
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    g = np.load(out)
    dec = D.unpack(g, 3, 4)
    assert [d["rank"] for d in dec] == [0, 1]
    for r, d in enumerate(dec):
        pi, pv, pc, tt, tr, tz, tc = (x.numpy() for x in _fake_results(r, 5, 3, 6, 0))
        assert d["event_base"] == 5 * r and d["n_events"] == 5
        assert d["pairs_grid"] == np.float32(1.5 * (r + 1)) * 1e9 and d["pairs_ms"] == np.float32(2.5) * 1e9
        assert np.array_equal(d["n_peaks"], pc) and np.array_equal(d["n_tracks"], tc)
        assert d["peaks_total"] == pc.sum() and d["tracks_total"] == tc.sum()
        for e in range(5):
            k = min(4, pc[e])
            assert np.array_equal(d["peak_index"][e, :k], pi[e, :k])
            assert np.all(d["peak_index"][e, k:] == -1)
            assert np.allclose(d["peak_value"][e, :k], pv[e, :k])
            kt = min(4, tc[e])
            assert np.allclose(d["tracks"][e, :kt, :3], tt[e, :kt])
            assert np.allclose(d["tracks"][e, :kt, 3], tr[e, :kt])
            assert np.array_equal(d["tracks"][e, :kt, 4], tz[e, :kt])
            assert np.all(d["tracks"][e, kt:] == 0)


def test_world_size_invariant_inputs():
    cfg = C.CFG3
    full = G.make_batch(cfg, range(8))
    for w in (2, 4, 8):
        parts = [G.make_batch(cfg, range(*D.shard(8, r, w))) for r in range(w)]
        hits = np.concatenate([p.hits for p in parts])
        assert np.array_equal(hits, full.hits)
