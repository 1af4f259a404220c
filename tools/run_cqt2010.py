"""Runs the CQT2010v2 forward a few times on the full 1,770-clip batch (for ncu)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1912_12055_b200.engine import Cqt2010Engine
from paper_1912_12055_b200.spectro import CqtConfig, cqt2010_plan

dev = torch.device("cuda:0")
p = cqt2010_plan(CqtConfig(sr=44100.0))
eng = Cqt2010Engine(p["taps"], p["top_kernels"], p["early_stages"], p["n_octaves"], p["kernel_hop"], p["first_bin"],
                    12, 84, "reflect", device=dev)
x = torch.randn(1770, 80000, device=dev) * 0.5
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    eng.forward(x)
torch.cuda.synchronize()
