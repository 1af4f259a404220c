"""Time CQT2010v2 (f16 chain) on the full batch and check it against the oracle on a few clips.
NNAB_CQT2010_MONO=1 selects the single fused kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.engine import Cqt2010Engine
cfg = O.CqtCfg(sr=44100.0)
p = O.cqt2010_plan(cfg)
eng = Cqt2010Engine(p.taps, p.top_kernels, p.early_stages, p.n_octaves, p.kernel_hop, p.first_bin, 12, 84, "reflect",
                    precision="f16")
x = torch.randn(1770, 80000, device="cuda") * 0.5
for _ in range(3): eng.forward(x)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): out = eng.forward(x)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
got = out.cpu().numpy()
xs = x.cpu().numpy()
errs = [O.peak_err(got[i], O.cqt2010v2_clip(xs[i].astype(np.float64), cfg, p)) for i in (0, 1, 777, 1769)]
print(f"mono={os.environ.get('NNAB_CQT2010_MONO', '0')} {ms:.3f} ms/batch = {659.8e6 / ms / 1e6:.0f} GB/s  errs {['%.2e' % e for e in errs]}")
