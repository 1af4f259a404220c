"""Per-octave / per-frame error map of the fused CQT2010v2 vs the oracle (debug)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.engine import Cqt2010Engine

cfg = O.CqtCfg(sr=44100.0)
p = O.cqt2010_plan(cfg)
rng = np.random.default_rng(1)
x = (rng.standard_normal((3, 80000)) * 0.5).astype(np.float32)
ref = np.stack([O.cqt2010v2_clip(c.astype(np.float64), cfg, p) for c in x])
eng = Cqt2010Engine(p.taps, p.top_kernels, p.early_stages, p.n_octaves, p.kernel_hop, p.first_bin, 12, 84, "reflect",
                    device="cuda:0")
got = eng.forward(torch.from_numpy(x).cuda()).cpu().numpy()
for i in range(3):
    pk = np.abs(ref[i]).max()
    d = np.abs(got[i] - ref[i]) / pk
    print(f"clip {i}: peak err {d.max():.2e}")
    for a in range(7):
        rows = slice(84 - 12 * (a + 1), 84 - 12 * a)
        da = d[rows]
        bad = np.where(da.max(axis=0) > 1e-3)[0]
        print(f"  octave {a}: max {da.max():.2e}  bad frames {bad[:8]}{'...' if len(bad) > 8 else ''} ({len(bad)})")
