"""CQT1992v2 operand modes: golden accuracy + full-batch timing (staging + GEMMs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.engine import CqtLongEngine
g = dict(np.load("tests/golden/golden.npz"))
cfg = O.CqtCfg(sr=44100.0)
kern, _ = O.cqt_time_bank(cfg)
xg = torch.from_numpy(g["clips"]).cuda()
xb = torch.randn(1770, 80000, device="cuda") * 0.5
for mode in ["tf32", "f16", "fp32", "3xtf32"]:
    e = CqtLongEngine(kern, 512, "reflect", precision=mode, device="cuda")
    got = e.forward(xg).cpu().numpy()
    err = max(O.peak_err(got[i], g["cqt1992v2_full"][i]) for i in range(2))
    for _ in range(3): e.forward(xb)
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    ts, tg = [], []
    for _ in range(10):
        a.record(); B, Ln = e.stage(xb); b.record(); e.run_staged(B, Ln); c.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b)); tg.append(b.elapsed_time(c))
    print(f"{mode:7s} prec={e.precision} err {err:.2e}  stage {np.median(ts):.3f} ms  gemms {np.median(tg):.3f} ms", flush=True)
