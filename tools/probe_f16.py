"""GPU probe: accuracy + timing of the STFT/Mel operand modes (tf32, 3xtf32, f16, 3xf16)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200 import _lib as L
from paper_1912_12055_b200.engine import DftEngine

g = dict(np.load("tests/golden/golden.npz"))
h_re, h_im = O.stft_bank()
W = O.mel_bank(44100.0, 2048, 128, formula="slaney")
x = torch.from_numpy(g["clips"]).cuda()
for mode in ["tf32", "3xtf32", "f16", "3xf16"]:
    e = DftEngine(h_re, h_im, 512, precision=mode, device="cuda")
    e.precision = L.PRECISIONS[mode]; e.set_bank(h_re, h_im)
    s = e.forward(x, "magnitude").cpu().numpy()
    es = max(O.peak_err(s[i], g["stft_mag_full"][i]) for i in range(2))
    e.set_mel(W)
    m = e.forward(x, "mel").cpu().numpy()
    em = max(O.peak_err(m[i], g["mel_full"][i]) for i in range(2))
    rng = np.random.default_rng(1)
    errs = []
    for amp in [1e-7, 1e-3, 1.0, 3e4]:
        xc = (rng.standard_normal((2, 20000)) * amp).astype(np.float32)
        got = e.forward(torch.from_numpy(xc).cuda(), "magnitude").cpu().numpy()
        ref = np.stack([O.stft_clip(c.astype(np.float64), h_re, h_im, 512) for c in xc])
        errs.append(max(O.peak_err(got[i], ref[i]) for i in range(2)))
    # timing at the full batch
    xb = torch.randn(1770, 80000, device="cuda") * 0.5
    for _ in range(3): e.forward(xb, "mel")
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    ts, tg = [], []
    for _ in range(10):
        a.record(); B, Ln = e.stage(xb); b.record(); e.run_staged(B, Ln, "mel"); c.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b)); tg.append(b.elapsed_time(c))
    print(f"{mode:7s} stft {es:.2e} mel {em:.2e} amps {['%.1e' % v for v in errs]}  stage {np.median(ts):.3f} ms  gemm {np.median(tg):.3f} ms  -> {2.406e12/np.median(tg)/1e9:.0f} TF/s", flush=True)
    del xb
