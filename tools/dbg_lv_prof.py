import sys, ctypes as C, os
sys.path.insert(0, ".")
import torch
from paper_1912_12055_b200 import _lib as L
from paper_1912_12055_b200.engine import Cqt2010Engine
from paper_1912_12055_b200.spectro import CqtConfig, cqt2010_plan
lib = L.load()
fn = lib.nnab_debug_cqt2010_profile
fn.restype = C.c_int; fn.argtypes = [C.c_int, C.c_void_p]
p = cqt2010_plan(CqtConfig(sr=44100.0))
eng = Cqt2010Engine(p["taps"], p["top_kernels"], p["early_stages"], p["n_octaves"], p["kernel_hop"], p["first_bin"], 12, 84, "reflect")
NB = int(sys.argv[1]) if len(sys.argv) > 1 else 1770
x = torch.randn(NB, 80000, device="cuda") * 0.5
eng.forward(x); torch.cuda.synchronize()
fn(1, None)
eng.forward(x); torch.cuda.synchronize()
out = (C.c_ulonglong * 16)()
fn(0, out)
n = max(out[5], 1)
for i, name in enumerate(["prologue", "build", "mma", "epilogue", "teardown"]):
    print(f"{name:10s} {out[i] / n / 1000:8.2f} us per CTA (sum over tiles)")
print("CTAs", out[5])
