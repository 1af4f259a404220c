"""Where does the FP32-mode joint mel+STFT kernel gradient error come from? (B clips)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200 import _lib as L
from paper_1912_12055_b200.layers import MelSpectrogram
B = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rng = np.random.default_rng(5)
x = (rng.standard_normal((B, 80000)) * 0.5).astype(np.float32)
h_re, h_im = O.stft_bank()
W = O.mel_bank(44100.0, 2048, 128, formula="slaney")
for fwd in ["3xf16", "3xtf32", "none"]:
    m = MelSpectrogram(sr=44100, trainable_mel=True, trainable_STFT=True, precision="fp32")
    op = m._op
    if fwd == "3xtf32":
        op.fwd_prec = L.PREC_3XTF32; op.fwd_engine.precision = L.PREC_3XTF32; op.fwd_engine.set_bank(h_re, h_im)
    elif fwd == "none":
        op.fwd_engine = None
    xt = torch.from_numpy(x).cuda()
    out = m(xt)
    g = np.random.default_rng(7).standard_normal(out.shape).astype(np.float32)
    out.backward(torch.from_numpy(g).cuda())
    dh_re = np.zeros_like(h_re); dh_im = np.zeros_like(h_im); dW = np.zeros_like(W)
    for b in range(B):
        fr, re, im, S = O.smooth_mag_forward(x[b].astype(np.float64), h_re, h_im, 512)
        gb = g[b].astype(np.float64); dS = W.T @ gb
        dW += gb @ S.T
        dh_re += (dS * re / S) @ fr; dh_im += (dS * im / S) @ fr
    gre, gim = m.h_re.grad.cpu().numpy(), m.h_im.grad.cpu().numpy()
    e_re = np.abs(gre - dh_re).max(axis=1) / np.abs(dh_re).max()
    e_im = np.abs(gim - dh_im).max(axis=1) / np.abs(dh_im).max()
    print(f"fwd={fwd:6s} B={B} dW {O.peak_err(m.mel_basis.grad.cpu().numpy(), dW):.2e} dh_re {e_re.max():.2e} (bin {e_re.argmax()}) dh_im {e_im.max():.2e} (bin {e_im.argmax()})  top im bins {np.argsort(e_im)[-5:]} {np.sort(e_im)[-5:]}")
