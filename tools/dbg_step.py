import sys
sys.path.insert(0, ".")
import torch
from paper_1912_12055_b200.layers import STFT
dev = torch.device("cuda:0")
m = STFT(n_fft=256, hop_length=64, sr=8000, trainable=True, precision="fp32")
x = torch.randn(4, 4000, device=dev)
opt = torch.optim.SGD(m.parameters(), lr=1e-3)
a = m(x).sum()
a.backward()
opt.step()
b = m(x).sum()
print("no-sync", float(a), float(b), m.h_re._version, m._op._bank_version)
