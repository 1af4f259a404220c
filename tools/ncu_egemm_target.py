"""E-GEMM CQT1992v2 forward on the lowest `n` bins (default 12), for ncu captures:
    python tools/ncu_egemm_target.py [n_bins] [reps]"""
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_1912_12055_b200 import banks
from paper_1912_12055_b200.engine import CqtLongEngine
from paper_1912_12055_b200.spectro import CqtConfig

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
k, _ = banks.cqt_time_kernels(bench.SR, CqtConfig(sr=bench.SR).bin_freqs_hz, 12, "hann", 1)
eng = CqtLongEngine(k[:n], 512, "reflect", device=dev, method="egemm")
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES, device=dev) * 0.5
for _ in range(reps):
    eng.forward(x)
torch.cuda.synchronize()
