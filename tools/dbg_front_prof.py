"""Per-role wait cycles of the CQT2010v2 front kernel (NNAB_CQT2010_LEVELS=3)."""
import ctypes as C, os, sys
os.environ["NNAB_CQT2010_LEVELS"] = "3"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200 import _lib as L
from paper_1912_12055_b200.engine import Cqt2010Engine
lib = L.load()
fn = lib.nnab_debug_cqt2010_front_profile
fn.restype = C.c_int; fn.argtypes = [C.c_int, C.c_void_p]
cfg = O.CqtCfg(sr=44100.0)
p = O.cqt2010_plan(cfg)
eng = Cqt2010Engine(p.taps, p.top_kernels, p.early_stages, p.n_octaves, p.kernel_hop, p.first_bin, 12, 84, "reflect",
                    precision="f16")
x = torch.randn(1770, 80000, device="cuda") * 0.5
eng.forward(x); torch.cuda.synchronize()
fn(1, None)
eng.forward(x); torch.cuda.synchronize()
out = (C.c_ulonglong * 24)()
fn(0, out)
ncta = 148
names = [("scan", ["conv_start"]), ("loader", ["ring_empty"]), ("mma", ["a_full", "s1_free", "s2_ready", "s2_free"]),
         ("conv", ["ex_ready", "a_empty", "ring_full"]), ("epi", ["s1_done", "E2 named_sync", "s2_done(s2)", "E2 tmem_ld"])]
print(f"elapsed {out[20] / ncta / 1e3:.1f} kcycles per CTA")
for r, (n, ws) in enumerate(names):
    print(n, "  ".join(f"{w} {out[4 * r + i] / ncta / 1e3:.1f}k" for i, w in enumerate(ws)))
tl = (C.c_longlong * 192)()
lib.nnab_debug_cqt2010_front_timeline.argtypes = [C.c_void_p]
lib.nnab_debug_cqt2010_front_timeline(tl)
print("CTA 0 timeline (kcycles): scan0 scan1 conv0 conv1 mmaS1 epiS1 mmaS2 epiS2 E2start E1(k,0) E1end syncd")
for k in range(12):
    print(k, " ".join(f"{tl[12 * k + e] / 1e3:7.1f}" for e in range(12)))
