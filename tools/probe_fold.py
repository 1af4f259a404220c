"""Gradient error of the trainable STFT layer with the Nyquist bin folded or not (fold changes nothing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.spectro import DftKernelBank, Signal, spectrogram_vjp, TrainableLayer
for prec in ["fp32", "tf32"]:
    for fold in [1, 0]:
        h_re, h_im = O.stft_bank(256, 8000.0)
        layer = TrainableLayer(DftKernelBank(h_re, h_im), hop=64, precision=prec)
        op = layer._op
        for e in (op.engine, op.fwd_engine):
            if e is None: continue
            e._fold_exact = False; e.fold = fold; e.set_bank(torch.as_tensor(h_re), torch.as_tensor(h_im))
        x = (np.random.default_rng(4).standard_normal(4096) * 0.5).astype(np.float32)
        S = layer.spectrogram(Signal(x, 8000.0)).cpu().numpy()
        c = np.random.default_rng(5).standard_normal(S.shape)
        got = spectrogram_vjp(Signal(x, 8000.0), layer, c)
        ref = O.conv_layer_vjp(x.astype(np.float64), h_re, h_im, 64, c)
        e_re = np.abs(got["h_re"].cpu().numpy() - ref["h_re"]).max(axis=1) / np.abs(ref["h_re"]).max()
        e_im = np.abs(got["h_im"].cpu().numpy() - ref["h_im"]).max(axis=1) / np.abs(ref["h_im"]).max()
        print(prec, "fold", fold, "re", e_re.max(), e_re.argmax(), "im", e_im.max(), e_im.argmax())
