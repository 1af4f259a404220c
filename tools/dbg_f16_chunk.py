"""Accuracy of the 3xF16 kernel-gradient GEMM alone vs float64 (torch on the GPU), for the
TMEM accumulation chunk in NNAB_RGEMM_F16_CHUNK (read once per process).
    NNAB_RGEMM_F16_CHUNK=8192 python tools/dbg_f16_chunk.py [B]
coef = g (re = 1, im = 0 makes coef_re = g / sqrt(1 + eps)), so dK_re = g_slots @ frames."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as Fn
from paper_1912_12055_b200 import _lib as L
from paper_1912_12055_b200.engine import DftEngine

B = int(sys.argv[1]) if len(sys.argv) > 1 else 600
n_fft, hop, F, Lx = 2048, 512, 1025, 80000
lib = L.load()
dev = torch.device("cuda")
torch.manual_seed(0)
x = torch.randn(B, Lx, device=dev) * 0.5
h = torch.zeros(F, n_fft)
eng = DftEngine(h, h, hop, True, "reflect", precision="3xf16", device=dev, allow_fold=False)
f = eng.frames(B, Lx)
ld = lib.nnab_slots_ld(C.byref(f))
T = eng.n_frames(Lx)
ws = torch.empty(lib.nnab_stft_workspace_bytes(C.byref(f), L.PREC_3XF16), dtype=torch.uint8, device=dev)
st = L.stream_handle(dev)
L.check(lib.nnab_stage_frames(C.byref(f), x.data_ptr(), L.PREC_3XF16, ws.data_ptr(), ws.numel(), st), "stage")
g = torch.randn(B, F, T, device=dev)
re = torch.ones(F, ld, device=dev)
im = torch.zeros(F, ld, device=dev)
c16 = [torch.empty(2 * F, ld, dtype=torch.float16, device=dev) for _ in range(2)]
rexp = torch.empty(2 * F + 1, dtype=torch.int32, device=dev)
L.check(lib.nnab_dft_coef_f16(C.byref(f), ws.data_ptr(), ws.numel(), L.PREC_3XF16, g.data_ptr(), re.data_ptr(),
                              im.data_ptr(), F,
                              T, ld, 0.0, c16[0].data_ptr(), c16[1].data_ptr(), rexp.data_ptr(), st), "coef")
dk = torch.empty(2 * F, n_fft, device=dev)
part = torch.empty(max(lib.nnab_rgemm_partial_bytes(2 * F, n_fft, ld, 0) // 4, 1), device=dev)
L.check(lib.nnab_kernel_grad_f16(C.byref(f), c16[0].data_ptr(), c16[1].data_ptr(), 2 * F, ld, rexp.data_ptr(),
                                 dk.data_ptr(), n_fft, ws.data_ptr(), ws.numel(), L.PREC_3XF16, part.data_ptr(), 0, st),
        "dk")
torch.cuda.synchronize()
xp = Fn.pad(x.double()[:, None], (n_fft // 2, n_fft // 2), mode="reflect")[:, 0]
fr = xp.unfold(1, n_fft, hop)[:, :T]  # (B, T, n_fft)
ref = torch.einsum("bft,btn->fn", g.double(), fr)
err = float((dk[:F].double() - ref).abs().max() / ref.abs().max())
print(f"chunk {os.environ.get('NNAB_RGEMM_F16_CHUNK', 'default')} B={B} K={B * T}: dK peak err {err:.2e}, "
      f"im rows max {float(dk[F:].abs().max()):.1e}")
