"""Kernel-gradient error: the FP16 dK (default; 3xF16 in FP32 mode, one FP16 pass in TF32 mode) vs
the 3xTF32 / TF32 dK (NNAB_F16_DK=0).
    python tools/dbg_f16_dk.py [B] [precision: fp32|tf32]
Cases: the joint mel + STFT layer on N(0, 0.25) clips; the same with per-clip loudness
spread over 1e-3..1e3 and upstream grads scaled by 1e-9 (the scale logic's stress case)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.layers import MelSpectrogram

B = int(sys.argv[1]) if len(sys.argv) > 1 else 6
PREC = sys.argv[2] if len(sys.argv) > 2 else "fp32"
h_re, h_im = O.stft_bank()
W = O.mel_bank(44100.0, 2048, 128, formula="slaney")
for case in ["plain", "stress"]:
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((B, 80000)) * 0.5).astype(np.float32)
    gs = 1.0
    if case == "stress":
        x *= np.logspace(-3, 3, B).astype(np.float32)[:, None]
        gs = 1e-9
    ref = None
    for f16 in ["1", "0"]:
        os.environ["NNAB_F16_DK"] = f16
        m = MelSpectrogram(sr=44100, trainable_mel=True, trainable_STFT=True, precision=PREC)
        assert m._op.f16_dk == (f16 == "1")
        out = m(torch.from_numpy(x).cuda())
        g = (np.random.default_rng(7).standard_normal(out.shape) * gs).astype(np.float32)
        out.backward(torch.from_numpy(g).cuda())
        if ref is None:
            dh_re = np.zeros_like(h_re); dh_im = np.zeros_like(h_im)
            for b in range(B):
                fr, re, im, S = O.smooth_mag_forward(x[b].astype(np.float64), h_re, h_im, 512)
                dS = W.T @ g[b].astype(np.float64)
                dh_re += (dS * re / S) @ fr; dh_im += (dS * im / S) @ fr
            ref = (dh_re, dh_im)
        e_re = O.peak_err(m.h_re.grad.cpu().numpy(), ref[0])
        e_im = O.peak_err(m.h_im.grad.cpu().numpy(), ref[1])
        print(f"{PREC} {case:6s} B={B} f16_dk={f16}: dh_re {e_re:.2e} dh_im {e_im:.2e}", flush=True)
