"""Trainable CQT1992v2 (BASELINE config 3 bank, layers.CQT1992v2(trainable=True)) forward + backward
on the full 1,770 x 80,000 batch: ms per step and algorithmic TFLOP/s.

Algorithmic work: forward 4 M sum(N_k) (re and im of every bin over its own support) plus the
kernel gradients 4 M sum(N_k) = 8.9e11 FLOP per batch (M = 277,890 frames, sum N_k = 400,975).
    python tools/time_cqt_train.py [precision] [clips]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_12055_b200.layers import CQT1992v2

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1770
dev = torch.device("cuda:0")
m = CQT1992v2(sr=44100, hop_length=512, fmin=32.70, n_bins=84, bins_per_octave=12, trainable=True, precision=prec)
x = torch.randn(nb, 80000, device=dev) * 0.5
g = torch.randn(nb, 84, 157, device=dev) * 1e-3


def step():
    m.k_re.grad = m.k_im.grad = None
    m(x).backward(g)


for _ in range(2):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
n = 5
for _ in range(n):
    step()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / n
lens = m.lengths
flop = 8.0 * nb * 157 * float(lens.sum())
print(f"trainable CQT1992v2 {prec}: {ms:.2f} ms/step ({nb} clips), {flop / ms / 1e9:.1f} TFLOP/s algorithmic, "
      f"{nb / (ms / 1e3):.0f} spectrograms/s")
