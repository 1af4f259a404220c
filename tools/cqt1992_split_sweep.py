"""Sweep the hybrid's long-bin threshold (CqtLongEngine.LONG_HOPS) on the full batch."""
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_1912_12055_b200 import banks
from paper_1912_12055_b200.engine import CqtLongEngine
from paper_1912_12055_b200.spectro import CqtConfig

dev = torch.device("cuda:0")
k, lens = banks.cqt_time_kernels(bench.SR, CqtConfig(sr=bench.SR).bin_freqs_hz, 12, "hann", 1)
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES, device=dev) * 0.5
for hops in [int(a) for a in sys.argv[1:]] or [3, 4, 6, 8, 11, 16, 24]:
    CqtLongEngine.LONG_HOPS = hops
    e = CqtLongEngine(k, 512, "reflect", device=dev)
    for _ in range(2):
        e.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        e.forward(x)
    e1.record()
    torch.cuda.synchronize()
    n_long = e.hybrid[-1] if e.hybrid is not None else (84 if e.egemm is not None else 0)
    n_groups = e.hybrid[0][4] if e.hybrid is not None else None
    print(f"LONG_HOPS={hops:3d} n_long={n_long:3d} groups={n_groups} {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
