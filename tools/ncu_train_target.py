"""One trainable STFT+Mel forward/backward on the full batch (for ncu captures):
    python tools/ncu_train_target.py [reps] [phasor: split|tf32] [precision: tf32|fp32]"""
import sys
sys.path.insert(0, ".")
import torch
import bench
dev = torch.device("cuda:0")
step = bench.TrainStep(dev, sys.argv[3] if len(sys.argv) > 3 else "tf32", 1,
                        phasor=sys.argv[2] if len(sys.argv) > 2 else "split")
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES, device=dev) * 0.5
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    step.forward(x)
torch.cuda.synchronize()
