"""End-to-end (pinned host in -> device -> host out) Mel time per batch vs the pipeline's chunk size.
    python tools/e2e_chunks.py [chunk ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda:0")
eng, kind, work, _ = bench.build_workload("mel", dev, "f16")
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES) * 0.5
xh = x.pin_memory()
oh = torch.empty(bench.B_CLIPS, 128, bench.T_FRAMES, dtype=torch.float32, pin_memory=True)
for ch in [int(a) for a in sys.argv[1:]] or [30, 59, 118, 177]:
    for _ in range(2):
        eng.forward_host(xh, kind, chunk_clips=ch, out_host=oh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        eng.forward_host(xh, kind, chunk_clips=ch, out_host=oh)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunk {ch:4d}: {ms:.3f} ms/batch, {bench.B_CLIPS / ms * 1e3:.0f} spectrograms/s, "
          f"H2D {bench.B_CLIPS * bench.L_SAMPLES * 4 / ms / 1e6:.1f} GB/s", flush=True)
