"""Scratch timing of the STFT/Mel forward on the full 1,770-clip config."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import spectro_oracle as O
from paper_1912_12055_b200.engine import DftEngine

dev = torch.device("cuda:0")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1770
x = (torch.randn(B, 80000, device=dev) * 0.5)
h_re, h_im = O.stft_bank()
for prec in ["tf32", "fp32"]:
    eng = DftEngine(h_re, h_im, 512, precision=prec, device=dev)
    eng.set_mel(O.mel_bank(44100.0, 2048, 128, formula="slaney"))
    for kind in ["magnitude", "mel"]:
        for _ in range(3): eng.forward(x, kind)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        n = 5
        for _ in range(n): eng.forward(x, kind)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        flops = 2 * B * 157 * 2048 * 2050
        print(f"{prec} {kind}: {ms:.3f} ms  {flops/ms/1e9:.1f} TFLOP/s", flush=True)
