"""SURVEY.md §8(e) on one GPU: the per-event results of the whole pass do not depend on how the
batch is split (so any rank layout gives bit-identical tracks), and the device-written result
record (retina_pack_results) is the layout tests/pack_ref.py states, word for word."""
import numpy as np
import pytest
import torch

from paper_1709_08610_b200 import dist as D
from paper_1709_08610_b200.pipeline import RetinaPipeline, upload
from synth import configs as C
from synth import events as G
from tests.pack_ref import pack_ref

pytestmark = pytest.mark.gpu


def _run(cfg, ids, chunk=4, ms_algorithm=0):
    import bench
    b = G.make_batch(cfg, ids)
    sd = G.make_seeds(cfg, ids)
    spec = bench.make_spec(cfg)
    spec.ms_algorithm = ms_algorithm
    pipe = RetinaPipeline(spec, len(ids), chunk_events=chunk)
    pipe.run(upload(b.offsets, b.hits, sd))
    torch.cuda.synchronize()
    return pipe


def _event_outputs(pipe, e):
    pc, tc = int(pipe.peak_cnt[e]), int(pipe.t_count[e])
    kp, kt = min(pc, pipe.peak_idx.shape[1]), min(tc, pipe.t_seed.shape[1])
    return [np.array([pc, tc]), pipe.peak_idx[e, :kp].cpu().numpy(), pipe.peak_val[e, :kp].cpu().numpy(),
            pipe.peak_theta[e, :kp].cpu().numpy(), pipe.theta[e].cpu().numpy(), pipe.resp[e].cpu().numpy(),
            pipe.t_seed[e, :kt].cpu().numpy(), pipe.t_size[e, :kt].cpu().numpy(), pipe.t_theta[e, :kt].cpu().numpy(),
            pipe.t_resp[e, :kt].cpu().numpy()]


@pytest.mark.parametrize("name,E,seeds,splits", [("cfg3", 12, 2048, (5, 12)), ("cfg4", 4, 1024, (1, 3, 4)),
                                                 ("cfg2", 9, 4096, (4, 9))])
def test_pipeline_results_independent_of_the_event_split(name, E, seeds, splits):
    cfg = C.CONFIGS[name].replace(n_seeds=seeds)
    whole = _run(cfg, range(E))
    ref = [_event_outputs(whole, e) for e in range(E)]
    lo = 0
    for hi in splits:  # the batch [0, E) as consecutive rank shards [lo, hi)
        part = _run(cfg, range(lo, hi), chunk=3)
        for e in range(lo, hi):
            for a, b in zip(_event_outputs(part, e - lo), ref[e]):
                assert np.array_equal(a, b), (name, e)
        lo = hi
    assert sum(int(x[0][1]) for x in ref) >= 0


@pytest.mark.parametrize("name,E,seeds", [("cfg3", 6, 8192), ("cfg2", 5, 4096)])
def test_pipeline_culled_multistart_gives_the_dense_results(name, E, seeds):
    """The whole pass with the culled multi-start kernel (RETINA_MS_CULLED) gives every per-event
    output of the dense pass bit for bit: seeds' end points and responses, and therefore the tracks."""
    cfg = C.CONFIGS[name].replace(n_seeds=seeds)
    dense = _run(cfg, range(E))
    culled = _run(cfg, range(E), ms_algorithm=1)
    for e in range(E):
        for a, b in zip(_event_outputs(dense, e), _event_outputs(culled, e)):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (name, e)


def test_pack_kernel_matches_the_stated_layout():
    cfg = C.CFG2.replace(n_seeds=1024, axes=((-0.3, 0.3, 64), (-0.3, 0.3, 64)))
    E = 6
    pipe = _run(cfg, range(E))
    for keep in (0, 3, 64):
        hdr = D.header_words(1, 600, E, 1.25e10, 3.5e11)
        out = D.pack(pipe.peak_idx[:E], pipe.peak_val[:E], pipe.peak_cnt[:E], pipe.t_theta[:E], pipe.t_resp[:E],
                     pipe.t_size[:E], pipe.t_count[:E], keep, hdr)
        torch.cuda.synchronize()
        ref = pack_ref(*(x[:E].cpu().numpy() for x in (pipe.peak_idx, pipe.peak_val, pipe.peak_cnt, pipe.t_theta,
                                                         pipe.t_resp, pipe.t_size, pipe.t_count)), keep, hdr)
        assert np.array_equal(out.cpu().numpy(), ref), keep
        dec = D.unpack(out.cpu().numpy()[None], 2, keep)[0]
        assert dec["rank"] == 1 and dec["event_base"] == 600 and dec["n_events"] == E
        assert dec["peaks_total"] == int(pipe.peak_cnt[:E].sum()) and dec["pairs_ms"] == np.float32(350.0) * 1e9
    with pytest.raises(ValueError):  # a wrongly sized output buffer is rejected before the kernel
        D.pack(pipe.peak_idx[:E], pipe.peak_val[:E], pipe.peak_cnt[:E], pipe.t_theta[:E], pipe.t_resp[:E],
               pipe.t_size[:E], pipe.t_count[:E], 3, hdr, out=torch.empty(5, dtype=torch.int32, device="cuda"))
