"""Input-gradient error (all-ones upstream) of the TF32 / 3xTF32 STFT layer over random inputs."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.layers import STFT
dev = torch.device("cuda:0")
h_re, h_im = O.stft_bank(128, 8000.0)
for prec in ("tf32", "fp32"):
    m2 = STFT(n_fft=128, hop_length=32, sr=8000, precision=prec)
    errs = []
    for seed in range(40):
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        xr = torch.randn(2, 1000, device=dev, generator=g).requires_grad_(True)
        m2(xr).sum().backward()
        ref = np.stack([O.conv_layer_vjp(c.astype(np.float64), h_re, h_im, 32, np.ones((65, 1000 // 32 + 1)),
                                         with_input_grad=True)[1] for c in xr.detach().cpu().numpy()])
        errs.append(O.peak_err(xr.grad.cpu().numpy(), ref))
    e = np.array(errs)
    print(prec, "median %.2e  p90 %.2e  max %.2e" % (np.median(e), np.quantile(e, 0.9), e.max()))
