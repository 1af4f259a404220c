"""Print peak-normalised errors of every forward mode vs the float64 golden."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import spectro_oracle as O
from paper_1912_12055_b200.engine import DftEngine
g = dict(np.load("tests/golden/golden.npz"))
x = torch.from_numpy(g["clips"]).cuda()
h_re, h_im = O.stft_bank()
W = O.mel_bank(44100.0, 2048, 128, formula="slaney")
for prec in ["tf32", "fp32"]:
    e = DftEngine(h_re, h_im, 512, precision=prec)
    e.set_mel(W, 1.0)
    m = e.forward(x, "magnitude").cpu().numpy()
    print(prec, "stft", [O.peak_err(m[i], g["stft_mag_full"][i]) for i in range(2)])
    print(prec, "mel p1", [O.peak_err(e.forward(x, "mel").cpu().numpy()[i], g["mel_full"][i]) for i in range(2)])
    e.set_mel(W, 2.0)
    print(prec, "mel p2", [O.peak_err(e.forward(x, "mel").cpu().numpy()[i], g["mel_full_p2"][i]) for i in range(2)])
