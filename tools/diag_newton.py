import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import oracle as ora
from synth import configs as C, events as G
from tests import parity_util as PU
import paper_1709_08610_b200 as R
np.set_printoptions(linewidth=200, precision=3)
for name, S, ev in (("cfg2", 512, [0, 1, 2, 3]), ("cfg3", 512, [0, 1]), ("cfg4", 256, [0])):
    cfg = C.CONFIGS[name]
    b = G.make_batch(cfg, ev); seeds = G.make_seeds(cfg, ev, n_seeds=S)
    sig, eta, fsig, mh = C.newton_schedule(cfg)
    th, Rg, _, ne = R.retina_multistart_newton_ex(R.Events.from_numpy(b.offsets, b.hits), cfg.model, torch.from_numpy(seeds).cuda(), sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi)
    torch.cuda.synchronize(); th = th.cpu().numpy(); Rg = Rg.cpu().numpy(); ne = ne.cpu().numpy()
    rth, rR, _, m, rne, log = ora.newton(cfg.model, b.offsets, b.hits, seeds, sig, eta, fsig, mh, cfg.box_lo, cfg.box_hi, want_margin=True, want_evals=True, log_len=96)
    ranges = np.array(cfg.box_hi) - np.array(cfg.box_lo)
    dev = np.max(np.abs(th - rth) / ranges, axis=2)
    bad = (dev > 1e-3) | (ne != rne)
    print(name, "bad", bad.sum())
    for e, s in np.argwhere(bad)[:12]:
        lg = log[e, s]; lg = lg[lg >= 0]
        # per-step R of oracle along the path
        print(f" ({e},{s}) dev {dev[e,s]:.2e} evals gpu {ne[e,s]} ref {rne[e,s]} Rgpu {Rg[e,s]:.4g} Rref {rR[e,s]:.4g} nd {len(lg)} margins {lg[:24]}")
