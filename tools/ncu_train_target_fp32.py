"""One trainable STFT+Mel forward/backward in 3xTF32 (FP32-accurate) mode, for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import torch
import bench
dev = torch.device("cuda:0")
step = bench.TrainStep(dev, "fp32", 1)
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES, device=dev) * 0.5
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    step.forward(x)
torch.cuda.synchronize()
