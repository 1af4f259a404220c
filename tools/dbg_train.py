import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.layers import STFT, MelSpectrogram
dev = torch.device("cuda:0")
m = STFT(n_fft=256, hop_length=64, sr=8000, trainable=True, precision="fp32")
x = torch.randn(4, 4000, device=dev)
opt = torch.optim.SGD(m.parameters(), lr=1e-3)
a = m(x).sum(); a.backward()
print("grad norms", m.h_re.grad.norm().item(), m.h_im.grad.norm().item(), "ver", m.h_re._version)
h0 = m.h_re.detach().clone()
opt.step()
print("param delta", (m.h_re.detach() - h0).abs().max().item(), "ver", m.h_re._version)
b = m(x).sum()
print("a b", float(a), float(b))
for prec in ["tf32", "fp32"]:
    rng = np.random.default_rng(5); B = 6
    xx = (rng.standard_normal((B, 80000)) * 0.5).astype(np.float32)
    mm = MelSpectrogram(sr=44100, trainable_mel=True, trainable_STFT=True, precision=prec)
    out = mm(torch.from_numpy(xx).to(dev))
    g = rng.standard_normal(out.shape).astype(np.float32)
    out.backward(torch.from_numpy(g).to(dev))
    h_re, h_im = O.stft_bank(); W = O.mel_bank(44100.0, 2048, 128, formula="slaney")
    dW = np.zeros_like(W); dre = np.zeros_like(h_re); dim = np.zeros_like(h_im); fw = []
    for i in range(B):
        fr, re, im, S = O.smooth_mag_forward(xx[i].astype(np.float64), h_re, h_im, 512)
        fw.append(W @ S); gb = g[i].astype(np.float64); dW += gb @ S.T; dS = W.T @ gb
        dre += (dS * re / S) @ fr; dim += (dS * im / S) @ fr
    print(prec, "fwd", O.peak_err(out.detach().cpu().numpy(), np.stack(fw)), "dW", O.peak_err(mm.mel_basis.grad.cpu().numpy(), dW),
          "dre", O.peak_err(mm.h_re.grad.cpu().numpy(), dre), "dim", O.peak_err(mm.h_im.grad.cpu().numpy(), dim))
