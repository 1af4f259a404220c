"""CQT1992v2 split experiment: E-GEMM (hop-offset GEMM) for the lowest bins,
per-K-block schedule for the rest on a narrower (re-centred) bank; times both
and checks the union against the all-schedule output."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_1912_12055_b200 import banks
from paper_1912_12055_b200.engine import CqtLongEngine
from paper_1912_12055_b200.spectro import CqtConfig

dev = torch.device("cuda:0")
cfg = CqtConfig(sr=bench.SR)
k, lens = banks.cqt_time_kernels(bench.SR, cfg.bin_freqs_hz, 12, "hann", 1)
W = k.shape[1]
x = torch.randn(bench.B_CLIPS, bench.L_SAMPLES, device=dev) * 0.5


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


full = CqtLongEngine(k, 512, "reflect", device=dev)
t_full, ref = timed(lambda: full.forward(x))
print(f"schedule all 84 bins (W={W}): {t_full:.3f} ms", flush=True)
eg = CqtLongEngine(k, 512, "reflect", device=dev, method="egemm")
t_eg, o_eg = timed(lambda: eg.forward(x))
print(f"egemm all 84 bins: {t_eg:.3f} ms  err {((o_eg - ref).abs().max() / ref.abs().max()).item():.2e}", flush=True)
for ks in (12, 24, 36):
    lo = CqtLongEngine(k[:ks], 512, "reflect", device=dev, method="egemm")
    w2 = int(lens[ks]) + 2 + (int(lens[ks]) & 1)
    w2 += w2 & 1
    c0 = W // 2 - w2 // 2
    hi = CqtLongEngine(k[ks:, c0:c0 + w2], 512, "reflect", device=dev)
    t_lo, o_lo = timed(lambda: lo.forward(x))
    t_hi, o_hi = timed(lambda: hi.forward(x))
    e_lo = ((o_lo - ref[:, :ks]).abs().max() / ref.abs().max()).item()
    e_hi = ((o_hi - ref[:, ks:]).abs().max() / ref.abs().max()).item()
    print(f"split {ks}: egemm low {t_lo:.3f} ms (err {e_lo:.1e}, egemm={lo.egemm is not None}), "
          f"schedule high W'={w2} {t_hi:.3f} ms (err {e_hi:.1e}) -> {t_lo + t_hi:.3f} ms", flush=True)
    lo2 = CqtLongEngine(k[:ks], 512, "reflect", device=dev)
    t_lo2, _ = timed(lambda: lo2.forward(x))
    print(f"          schedule low {t_lo2:.3f} ms", flush=True)
