"""Bit-exact framing / padding on the hot path: the hop-row staging kernel
(`stage_rows_kernel`, csrc/frames.cu) that feeds every STFT / Mel / CQT1992v2
GEMM and the training dK GEMM, called through the C ABI (`nnab_stage_frames`).

The reference pads with np.pad (signal.py:138-156) and frames with
sliding_window_view (signal.py:181); its pad index map is pinned by the golden
vectors the reference produced (gradients.py:18-25: padmap_*).  Staging
x[b, i] = b*L + i + 1 in 3xTF32 mode stores each sample as TF32 hi + lo, which
is exact for integers below 2^22, so hi + lo recovers the source index of every
staged element: the staged rows must equal the index map exactly (0 for a zero
pad and beyond the padded clip).  The (L, pad) cases run all four load branches
of the kernel: aligned float4 interior, funnel-shifted unaligned interior
(pad or L not a multiple of 4), reversed-funnel reflected groups and the scalar
edges; several clips per batch put clip starts off 16-byte boundaries."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import spectro_oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # (L, width, hop, pad, mode, golden index-map key or None)
    (80000, 2048, 512, 1024, "reflect", "padmap_reflect_80000_1024"),      # STFT / Mel (BASELINE 1, 2)
    (80000, 22682, 512, 11341, "reflect", "padmap_reflect_80000_11341"),  # CQT1992v2 (BASELINE 3)
    (100, 14, 32, 7, "constant_zero", "padmap_zero_100_7"),               # width < hop, zero pad
    (1001, 64, 32, 13, "reflect", None),     # L, pad odd: unaligned clip starts + funnels
    (4099, 256, 64, 131, "reflect", None),   # hop rows, pad % 4 == 3
    (998, 74, 37, 37, "reflect", None),      # hop % 32 != 0: rows are whole frames (row_len = 96)
    (5003, 512, 128, 254, "constant_zero", None),
]


def _stage(x: torch.Tensor, width, hop, pad, mode):
    from paper_1912_12055_b200 import _lib as L
    from paper_1912_12055_b200.engine import frames_struct
    lib = L.load()
    B, n = x.shape
    f = frames_struct(B, n, width, hop, pad, mode)
    T, rl, R = C.c_int32(), C.c_int32(), C.c_int32()
    L.check(lib.nnab_frames_geometry(C.byref(f), C.byref(T), C.byref(rl), C.byref(R)), "geometry")
    nbytes = lib.nnab_stft_workspace_bytes(C.byref(f), L.PREC_3XTF32)
    ws = torch.zeros(nbytes // 4, dtype=torch.float32, device=x.device)
    L.check(lib.nnab_stage_frames(C.byref(f), x.data_ptr(), L.PREC_3XTF32, ws.data_ptr(), nbytes,
                                  L.stream_handle(x.device)), "stage_frames")
    torch.cuda.synchronize()
    rows = B * R.value * rl.value
    half = nbytes // 8  # hi then lo, each stage_bytes (256-aligned)
    hi = ws[:rows].double().cpu().numpy()
    lo = ws[half:half + rows].double().cpu().numpy()
    return (hi + lo).reshape(B, R.value, rl.value), T.value, rl.value, R.value


@pytest.mark.parametrize("n,width,hop,pad,mode,key", CASES)
def test_staged_rows_equal_index_map(golden, cuda_dev, n, width, hop, pad, mode, key):
    B = 3
    x = (np.arange(B)[:, None] * n + np.arange(n)[None, :] + 1).astype(np.float32)
    assert x.max() < 2 ** 22
    got, T, rl, R = _stage(torch.from_numpy(x).to(cuda_dev), width, hop, pad, mode)
    imap = O.pad_index_map(n, pad, pad, mode)  # np.pad, the reference's own pad (signal.py:151)
    if key is not None:  # ... and pinned to the index map the reference itself produced
        want_map = golden[key].astype(np.int64)
        if mode == "constant_zero":
            want_map = np.where(want_map < 0, -1, want_map)
        assert np.array_equal(imap, want_map)
    padded_len = n + 2 * pad
    assert T == (padded_len - width) // hop + 1
    for b in range(B):
        src = np.where(imap >= 0, b * n + imap + 1, 0).astype(np.float64)
        # hop rows (rl == hop): row r holds padded[r*hop, r*hop + hop); whole frames
        # (rl = width rounded up to 32): row t holds padded[t*hop, t*hop + rl), the
        # columns past `width` meeting the bank's zero K padding
        pos = np.arange(R)[:, None] * hop + np.arange(rl)[None, :]
        want = np.where(pos < padded_len, src[np.minimum(pos, padded_len - 1)], 0.0)
        assert np.array_equal(got[b], want), (b, np.argwhere(got[b] != want)[:5])
    # the frames the GEMM reads (hop rows t .. t + width/hop - 1) are the reference's
    # sliding_window_view frames of the padded clip (signal.py:181)
    if rl == hop and width % hop == 0:
        for b in (0, B - 1):
            src = np.where(imap >= 0, b * n + imap + 1, 0).astype(np.float64)
            frames = np.lib.stride_tricks.sliding_window_view(src, width)[::hop]
            flat = got[b].reshape(-1)
            for t in (0, 1, T // 2, T - 2, T - 1):
                assert np.array_equal(flat[t * hop:t * hop + width], frames[t])


def test_tf32_staging_rounds_to_nearest_even(cuda_dev):
    """TF32 mode stores RNE(x) to 10 mantissa bits (what the tensor core reads)."""
    from paper_1912_12055_b200 import _lib as L
    from paper_1912_12055_b200.engine import frames_struct
    lib = L.load()
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 4096)).astype(np.float32)
    f = frames_struct(2, 4096, 512, 128, 256, "reflect")
    nbytes = lib.nnab_stft_workspace_bytes(C.byref(f), L.PREC_TF32)
    ws = torch.zeros(nbytes // 4, dtype=torch.float32, device=cuda_dev)
    xd = torch.from_numpy(x).to(cuda_dev)
    L.check(lib.nnab_stage_frames(C.byref(f), xd.data_ptr(), L.PREC_TF32, ws.data_ptr(), nbytes,
                                  L.stream_handle(cuda_dev)), "stage_frames")
    torch.cuda.synchronize()
    T, rl, R = C.c_int32(), C.c_int32(), C.c_int32()
    lib.nnab_frames_geometry(C.byref(f), C.byref(T), C.byref(rl), C.byref(R))
    got = ws[: 2 * R.value * rl.value].cpu().numpy().reshape(2, -1)
    i = O.pad(x.astype(np.float64), 256, 256, "reflect").astype(np.float32).view(np.uint32)
    rne = ((i + 0xFFF + ((i >> 13) & 1)) & ~np.uint32(0x1FFF)).view(np.float32)
    n = min(got.shape[1], rne.shape[1])
    assert np.array_equal(got[:, :n], rne[:, :n])
