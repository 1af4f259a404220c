"""CPU tests: the C-ABI library loads and exports every symbol include/nnab.h
declares (no compute calls without a GPU), the host-side bank builders match
the oracle, host-side geometry/schedule logic, and that the product path
refuses to run without a B200 (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from oracle import spectro_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "nnab.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nnab_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1912_12055_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares a prototype for each of them
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_host_only_entry_points():
    from paper_1912_12055_b200 import _lib as L
    lib = L.load()
    assert lib.nnab_version() >= 1
    assert lib.nnab_strerror(L.EINVAL) == b"invalid argument"
    # geometry: 80,000 samples, n_fft 2048, hop 512, centred -> 157 frames, hop-row staging
    f = L.nnab_frames(1770, 80000, 2048, 512, 1024, L.PAD_REFLECT)
    t, rl, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.nnab_frames_geometry(ctypes.byref(f), ctypes.byref(t), ctypes.byref(rl), ctypes.byref(r)) == 0
    assert (t.value, rl.value, r.value) == (157, 512, 160)
    assert lib.nnab_slots_ld(ctypes.byref(f)) == 1770 * 160
    # CQT1992v2 geometry: width 22,682 padded by 11,341 -> 157 frames
    f2 = L.nnab_frames(2, 80000, 22682, 512, 11341, L.PAD_REFLECT)
    assert lib.nnab_frames_geometry(ctypes.byref(f2), ctypes.byref(t), ctypes.byref(rl), ctypes.byref(r)) == 0
    assert t.value == 157
    # reflect pad >= length -> EINVAL (signal.py:147-150)
    bad = L.nnab_frames(1, 100, 256, 64, 128, L.PAD_REFLECT)
    assert lib.nnab_frames_geometry(ctypes.byref(bad), None, None, None) == L.EINVAL
    # bank tiles: default 1025 bins fold into exactly 8 tiles
    assert lib.nnab_dft_bank_tiles(1025, 1) == 8 and lib.nnab_dft_bank_tiles(1025, 0) == 9
    assert lib.nnab_stft_workspace_bytes(ctypes.byref(f), L.PREC_TF32) == 1770 * 160 * 512 * 4


def test_cqt_schedule_is_longest_first_prefix():
    from paper_1912_12055_b200 import _lib as L
    from paper_1912_12055_b200 import banks
    from paper_1912_12055_b200.engine import _row_support
    from paper_1912_12055_b200.spectro import CqtConfig
    lib = L.load()
    cfg = CqtConfig(sr=44100.0)
    k, lens = banks.cqt_time_kernels(cfg.sr, cfg.bin_freqs_hz, 12, "hann", 1)
    sup = _row_support(k.real.astype(np.float32), k.imag.astype(np.float32))
    assert np.all(sup[:, 1] - sup[:, 0] <= lens + 1)
    tab = np.zeros(2000, dtype=np.uint32)
    n = ctypes.c_int32()
    assert lib.nnab_cqt_schedule(sup.ctypes.data, 84, k.shape[1], L.PREC_TF32, tab.ctypes.data, ctypes.byref(n)) == 0
    ent = tab[: n.value]
    widths = ent & 0xFFFF
    assert widths[0] == 176 and np.all(np.diff(widths.astype(int)) <= 0)
    # executed MMA rows x K vs dense: the schedule skips the zero support
    assert widths.sum() * 32 < 0.3 * 176 * k.shape[1]
    # every K block touching any kernel is scheduled exactly once
    kbs = ent >> 16
    assert len(set(kbs.tolist())) == len(kbs)


def test_host_banks_match_oracle():
    from paper_1912_12055_b200 import banks
    nf, hz = banks.frequency_scale("no", 2048, 44100.0, 50.0, 6000.0, None)
    h_re, h_im = banks.dft_kernels(nf, banks.make_window("hann", 2048, True))
    o_re, o_im = O.stft_bank()
    assert np.array_equal(h_re, o_re) and np.array_equal(h_im, o_im)
    for formula, norm in [("slaney", "none"), ("htk", "area")]:
        w, _ = banks.mel_filter_bank(44100.0, 2048, 128, formula=formula, norm=norm)
        assert np.allclose(w, O.mel_bank(44100.0, 2048, 128, formula=formula, norm=norm), atol=1e-15)
    for kind in ("linear", "log"):
        nf, _ = banks.frequency_scale(kind, 256, 8000.0, 80.0, 3500.0, 100)
        assert np.allclose(nf, O.freq_ladder(kind, 256, 8000.0, 80.0, 3500.0, 100), rtol=1e-15)
    assert np.array_equal(banks.lowpass_fir(255, 0.5), O.lowpass_taps(255, 0.5))
    k, lens = banks.cqt_time_kernels(44100.0, O.CqtCfg(sr=44100.0).freqs(), 12, "hann", 1)
    ko, lo = O.cqt_time_bank(O.CqtCfg(sr=44100.0))
    assert np.array_equal(lens, lo) and np.allclose(k, ko, atol=1e-18)


def test_cqt2010_plan_matches_oracle():
    from paper_1912_12055_b200.spectro import CqtConfig, cqt2010_plan
    for kw in [dict(sr=44100.0), dict(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256),
               dict(sr=22050.0, fmin=82.0, n_bins=50, hop_length=256),
               dict(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256, early_downsample=False)]:
        p, q = cqt2010_plan(CqtConfig(**kw)), O.cqt2010_plan(O.CqtCfg(**kw))
        assert (p["n_octaves"], p["early_stages"], p["kernel_hop"], p["first_bin"]) == \
            (q.n_octaves, q.early_stages, q.kernel_hop, q.first_bin)
        assert np.allclose(p["top_kernels"], q.top_kernels, atol=1e-18)
    with pytest.raises(ValueError, match="divisible"):
        cqt2010_plan(CqtConfig(sr=22050.0, fmin=55.0, n_bins=48, hop_length=100))
    with pytest.raises(ValueError):
        CqtConfig(sr=8000.0, fmin=2000.0, n_bins=36)  # top bin above Nyquist (kernels.py:312-316)


def test_mel_bands_cover_nonzeros():
    from paper_1912_12055_b200 import banks
    w, _ = banks.mel_filter_bank(44100.0, 2048, 128, formula="slaney")
    band = banks.mel_bands(np.pad(w, ((0, 0), (0, 63))), 34)
    for c in range(33):
        nz = np.nonzero(w[:, c * 32:(c + 1) * 32].any(axis=1))[0]
        if nz.size:
            assert band[c, 0] <= nz[0] and band[c, 1] >= nz[-1] + 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_refuses_cpu():
    from paper_1912_12055_b200._lib import NnabError
    from paper_1912_12055_b200.engine import DftEngine
    h_re, h_im = O.stft_bank(256, 8000.0)
    with pytest.raises(NnabError):
        DftEngine(h_re, h_im, 64, device="cuda")
    with pytest.raises(NnabError):
        DftEngine(h_re, h_im, 64, device="cpu")


def test_shard_range():
    from paper_1912_12055_b200.dist import shard_range
    sizes = [shard_range(1770, r, 8) for r in range(8)]
    assert [hi - lo for lo, hi in sizes] == [222, 222, 221, 221, 221, 221, 221, 221]
    assert sizes[0][0] == 0 and sizes[-1][1] == 1770
    assert all(sizes[i][1] == sizes[i + 1][0] for i in range(7))
    with pytest.raises(ValueError):
        shard_range(10, 3, 3)


def test_wav_header_errors(tmp_path):
    """wavio.py:26-63 error behaviour, mirrored by the host-side parser (no GPU)."""
    import struct
    from paper_1912_12055_b200 import fileio
    bad = tmp_path / "bad.wav"
    bad.write_bytes(b"RIFX0000WAVE")
    with pytest.raises(fileio.CorruptFileError):
        fileio._parse_wav(str(bad))
    fmt = struct.pack("<HHIIHH", 1, 1, 8000, 24000, 3, 24)  # 24-bit PCM
    body = b"WAVE" + b"fmt " + struct.pack("<I", 16) + fmt + b"data" + struct.pack("<I", 6) + b"\x00" * 6
    w24 = tmp_path / "w24.wav"
    w24.write_bytes(b"RIFF" + struct.pack("<I", len(body)) + body)
    with pytest.raises(fileio.UnsupportedFormatError):
        fileio._parse_wav(str(w24))
    trunc = tmp_path / "t.wav"
    trunc.write_bytes(b"RIFF" + struct.pack("<I", 100) + b"WAVE" + b"data" + struct.pack("<I", 50) + b"\x00" * 10)
    with pytest.raises(fileio.CorruptFileError):
        fileio._parse_wav(str(trunc))
    assert issubclass(fileio.CorruptFileError, ValueError) and issubclass(fileio.UnsupportedFormatError, ValueError)


def test_fp16_kernel_gradient_argument_checks():
    """nnab_*_f16 reject bad arguments before touching a device: an unknown staging precision,
    a missing workspace, a 3xF16 kernel gradient over a one-pass (F16) staging."""
    from paper_1912_12055_b200 import _lib as L
    lib = L.load()
    f = L.nnab_frames(4, 80000, 2048, 512, 1024, L.PAD_REFLECT)
    ld = lib.nnab_slots_ld(ctypes.byref(f))
    fake = 1 << 20  # never dereferenced: every call below fails its checks first
    assert lib.nnab_kernel_grad_f16(ctypes.byref(f), fake, fake, 2050, ld, fake, fake, 2048, fake, 1 << 40,
                                    L.PREC_TF32, fake, 0, None) == L.EINVAL  # not an FP16 staging
    assert lib.nnab_kernel_grad_f16(ctypes.byref(f), fake, fake, 2050, ld, fake, fake, 2048, None, 0,
                                    L.PREC_3XF16, fake, 0, None) == L.EINVAL  # no workspace
    f16_bytes = lib.nnab_stft_workspace_bytes(ctypes.byref(f), L.PREC_F16)
    assert lib.nnab_kernel_grad_f16(ctypes.byref(f), fake, fake, 2050, ld, fake, fake, 2048, fake, f16_bytes,
                                    L.PREC_F16, fake, 0, None) == L.EINVAL  # lo rows needed, staging has none
    assert lib.nnab_dft_coef_f16(ctypes.byref(f), fake, 1 << 40, L.PREC_3XF16, None, fake, fake, 1025, 157, ld,
                                 1e-12, fake, fake, fake, None) == L.EINVAL  # no upstream grad
    assert lib.nnab_mel_dft_coef_f16(ctypes.byref(f), fake, 1 << 40, L.PREC_3XF16, 1025, ld, 128, fake, None, fake,
                                     fake, 128, fake, fake, 1e-12, fake, fake, fake, None) == L.EINVAL  # 3xTF32 w/o wt_lo
