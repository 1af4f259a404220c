"""Pair-mode reduction GEMM check + timing at the training dK shape.
Run twice: NNAB_RGEMM_PAIR=0 (single CTAs) and default (CTA pairs)."""
import sys, os
sys.path.insert(0, ".")
import torch
from paper_1912_12055_b200 import _lib as L
lib = L.load()
dev = torch.device("cuda:0")
torch.manual_seed(0)


def run(M, N, K, hop, splits=0, reps=5):
    A = torch.randn(M, K, device=dev)
    x = torch.randn(K * hop + N, device=dev)
    # B(k, n) = x[k * hop + n]: hop rows (MN-major, row length hop)
    c = torch.zeros(M, N, device=dev)
    part = torch.empty(lib.nnab_rgemm_partial_bytes(M, N, K, splits) // 4 + 1, device=dev)
    rows = (K * hop + N) // hop
    st = L.stream_handle(dev)
    f = lambda: lib.nnab_rgemm(M, N, K, A.data_ptr(), None, K, x.data_ptr(), None, 0, 1, hop, rows,
                               c.data_ptr(), N, splits, part.data_ptr(), 0, st)
    assert f() == 0
    torch.cuda.synchronize()
    # check a subset of columns in float64
    cols = torch.arange(0, N, 37, device=dev)
    idx = torch.arange(K, device=dev)[:, None] * hop + cols[None, :]
    ref = A.double() @ x.double()[idx]
    err = ((c[:, cols].double() - ref).abs().max() / ref.abs().max()).item()
    s = torch.cuda.Stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for _ in range(reps):
        f()
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K / ms / 1e9
    print(f"pair={os.environ.get('NNAB_RGEMM_PAIR', '1')} M={M} N={N} K={K} hop={hop} err={err:.2e} {ms:.3f} ms {tf:.0f} TF/s",
          flush=True)


run(2050, 2048, 283200, 512)
run(1000, 2048, 65536, 512)
run(1000, 1000, 70016, 480)
run(256, 512, 16384, 512)
run(300, 2048, 8192, 256)
