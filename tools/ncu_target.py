"""Runs one workload's forward a few times on the full 1,770-clip batch, for ncu
captures of its kernels:  python tools/ncu_target.py mel|stft|cqt1992v2|cqt2010v2 [reps] [mode]"""
import sys
sys.path.insert(0, ".")
import torch
import bench

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = sys.argv[3] if len(sys.argv) > 3 else "f16"
dev = torch.device("cuda:0")
eng, kind, work, _ = bench.build_workload(name, dev, mode)
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES, device=dev) * 0.5
for _ in range(reps):
    eng.forward(x, kind)
torch.cuda.synchronize()
