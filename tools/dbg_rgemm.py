import sys, ctypes as C
sys.path.insert(0, ".")
import torch
from paper_1912_12055_b200 import _lib as L
lib = L.load()
dev = torch.device("cuda:0")
torch.manual_seed(0)
def run(M, N, K, b_mn, prec=0, splits=1):
    A = torch.randn(M, K, device=dev)
    if b_mn:
        Bm = torch.randn(K, N, device=dev)     # (k, n) at rows[k][n]
        ref = A.double() @ Bm.double()
        b, ldb, rl, rows = Bm, 0, N, K
    else:
        Bm = torch.randn(N, K, device=dev)
        ref = A.double() @ Bm.double().T
        b, ldb, rl, rows = Bm, K, 0, 0
    c = torch.zeros(M, N, device=dev)
    part = torch.empty(lib.nnab_rgemm_partial_bytes(M, N, K, splits) // 4 + 1, device=dev)
    rc = lib.nnab_rgemm(M, N, K, A.data_ptr(), None, K, b.data_ptr(), None, ldb, b_mn, rl, rows, c.data_ptr(), N, splits, part.data_ptr(), prec, L.stream_handle(dev))
    torch.cuda.synchronize()
    err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
    print(f"M={M} N={N} K={K} b_mn={b_mn} splits={splits} rc={rc} err={err:.3e} cmax={c.abs().max().item():.3e} refmax={ref.abs().max().item():.3e}")
    if b_mn and err > 1e-2:
        # which pattern? compare c against ref with B transposed etc
        for name, r in [("B^T-as-K-major", A.double() @ Bm.double().reshape(N, K).T)]:
            print(name, ((c.double() - r).abs().max() / r.abs().max()).item())
        print(c[:4, :8]); print(ref[:4, :8])
run(128, 256, 64, 0)
run(128, 256, 64, 1)
run(256, 512, 1024, 1, splits=4)
run(34, 32, 512, 1, splits=0)
