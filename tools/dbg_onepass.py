"""TF32-mode training gradients against float64, split-precision phasor vs the one-pass forward
(FP16 forward + one-pass FP16 dK by default; NNAB_F16_DK=0: the TF32 forward and TF32 dK).
    python tools/dbg_onepass.py [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.layers import MelSpectrogram
B = int(sys.argv[1]) if len(sys.argv) > 1 else 6
x = (np.random.default_rng(5).standard_normal((B, 80000)) * 0.5).astype(np.float32)
h_re, h_im = O.stft_bank()
W = O.mel_bank(44100.0, 2048, 128, formula="slaney")
ref = None
for ph in ["split", "tf32"]:
    m = MelSpectrogram(sr=44100, trainable_mel=True, trainable_STFT=True, precision="tf32", grad_phasor=ph)
    out = m(torch.from_numpy(x).cuda())
    g = np.random.default_rng(7).standard_normal(out.shape).astype(np.float32)
    out.backward(torch.from_numpy(g).cuda())
    if ref is None:
        dr, di, dW, fw = np.zeros_like(h_re), np.zeros_like(h_im), np.zeros_like(W), []
        for b in range(B):
            fr, re, im, S = O.smooth_mag_forward(x[b].astype(np.float64), h_re, h_im, 512)
            gb = g[b].astype(np.float64)
            dS = W.T @ gb
            dW += gb @ S.T
            dr += (dS * re / S) @ fr
            di += (dS * im / S) @ fr
            fw.append(W @ S)
        ref = (np.stack(fw), dW, dr, di)
    print(f"F16_DK={os.environ.get('NNAB_F16_DK', '1')} phasor={ph}: fwd {O.peak_err(out.detach().cpu().numpy(), ref[0]):.2e}"
          f" dW {O.peak_err(m.mel_basis.grad.cpu().numpy(), ref[1]):.2e}"
          f" dh_re {O.peak_err(m.h_re.grad.cpu().numpy(), ref[2]):.2e} dh_im {O.peak_err(m.h_im.grad.cpu().numpy(), ref[3]):.2e}")
