"""Plain numpy statement of the retina_pack_results record layout (include/retina.h), used to
build CPU records for the gloo tests and to check the device kernel word for word."""
import struct

import numpy as np

HEADER = 8


def pack_ref(peak_idx, peak_val, peak_cnt, t_theta, t_resp, t_size, t_count, keep, header):
    peak_idx, peak_val, peak_cnt = (np.asarray(x) for x in (peak_idx, peak_val, peak_cnt))
    t_theta, t_resp, t_size, t_count = (np.asarray(x) for x in (t_theta, t_resp, t_size, t_count))
    E, pcap = peak_idx.shape
    _, tcap, P = t_theta.shape
    W = 2 + 2 * keep + keep * (P + 2)

    def bits(v):
        return struct.unpack("<i", struct.pack("<f", float(np.float32(v))))[0]

    words = [int(np.uint32(h).astype(np.int32)) for h in header]
    words[3] = int(peak_cnt.astype(np.int64).sum())
    words[4] = int(t_count.astype(np.int64).sum())
    for e in range(E):
        pc, tc = int(peak_cnt[e]), int(t_count[e])
        rec = [pc, tc]
        rec += [int(peak_idx[e, k]) if k < min(pc, pcap) else -1 for k in range(keep)]
        rec += [bits(peak_val[e, k]) if k < min(pc, pcap) else 0 for k in range(keep)]
        for k in range(keep):
            if k < min(tc, tcap):
                rec += [bits(v) for v in t_theta[e, k]] + [bits(t_resp[e, k]), int(t_size[e, k])]
            else:
                rec += [0] * (P + 2)
        assert len(rec) == W
        words += rec
    return np.array(words, dtype=np.int64).astype(np.uint32).view(np.int32)
