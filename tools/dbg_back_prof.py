"""Per-role wait cycles of the CQT2010v2 back-end kernel (per CTA)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200 import _lib as L
from paper_1912_12055_b200.engine import Cqt2010Engine
lib = L.load()
fn = lib.nnab_debug_cqt2010_back_profile
fn.restype = C.c_int; fn.argtypes = [C.c_int, C.c_void_p]
cfg = O.CqtCfg(sr=44100.0)
p = O.cqt2010_plan(cfg)
eng = Cqt2010Engine(p.taps, p.top_kernels, p.early_stages, p.n_octaves, p.kernel_hop, p.first_bin, 12, 84, "reflect",
                    precision="f16")
x = torch.randn(1770, 80000, device="cuda") * 0.5
eng.forward(x); torch.cuda.synchronize()
fn(1, None)
eng.forward(x); torch.cuda.synchronize()
out = (C.c_ulonglong * 32)()
fn(0, out)
n = 148
names = [("h-producer", ["cgrp_done", "lvl_ready", "h_empty"]), ("h-MMA", ["hd_empty", "h_full"]),
         ("c-producer", ["lvl_ready", "c_mma"]), ("c-MMA", ["c_full", "c_tfree"]), ("h-epilogue", ["hd_full", "tiles(incl wait)", "margins+copies"]),
         ("c-epilogue", ["c_mma"])]
print(f"elapsed {out[24] / n / 1e3:.1f}k cycles per CTA")
for r, (nm, ws) in enumerate(names):
    print(nm, "  ".join(f"{w} {out[4 * r + i] / n / 1e3:.1f}k" for i, w in enumerate(ws)))
