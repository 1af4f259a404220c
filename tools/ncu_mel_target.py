"""One full-batch Mel forward (1,770 x 80,000) for an ncu capture: python tools/ncu_mel_target.py [precision] [kind]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_12055_b200 import banks
from paper_1912_12055_b200.engine import DftEngine
prec = sys.argv[1] if len(sys.argv) > 1 else "f16"
kind = sys.argv[2] if len(sys.argv) > 2 else "mel"
nf, _ = banks.frequency_scale("no", 2048, 44100.0, 50.0, 6000.0, None)
h_re, h_im = banks.dft_kernels(nf, banks.make_window("hann", 2048, True))
e = DftEngine(h_re, h_im, 512, precision=prec, device="cuda")
w, _ = banks.mel_filter_bank(44100.0, 2048, 128, formula="slaney", norm="none")
e.set_mel(w)
x = torch.randn(1770, 80000, device="cuda") * 0.5
for _ in range(2):
    e.forward(x, kind)
torch.cuda.synchronize()
