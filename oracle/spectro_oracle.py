"""CPU ORACLE -- test infrastructure only, never a product path.

A float64 NumPy restatement of the `spectro` reference's waveform -> spectrogram
hot path (the package under /root/reference/pkg/src/spectro).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import this
module, and only as the checker / CPU baseline.  The shipped path
(`paper_1912_12055_b200`) must never import it.

Parity is pinned: `tests/golden/make_golden.py` imports the real reference in
the build container and stores its outputs under `tests/golden/`;
`tests/test_oracle_golden.py` checks every function here against them.

Every function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/spectro/`).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

# ----------------------------------------------------------------------------
# windows, padding, strided correlation, FIR, decimation      (signal.py)
# ----------------------------------------------------------------------------


def window(kind: str, n: int, periodic: bool = True) -> np.ndarray:
    """signal.py:106-135 -- hann/hamming/blackman/rectangular, clipped to [0,1]."""
    if n < 1:
        raise ValueError("window length must be >= 1")
    if kind == "rectangular":
        return np.ones(n)
    if kind not in ("hann", "hamming", "blackman"):
        raise ValueError(f"unknown window kind {kind!r}")
    d = n if periodic else n - 1
    if d == 0:
        return np.ones(1)
    ph = 2.0 * np.pi * np.arange(n) / d
    if kind == "hann":
        v = 0.5 - 0.5 * np.cos(ph)
    elif kind == "hamming":
        v = 0.54 - 0.46 * np.cos(ph)
    else:
        v = 0.42 - 0.5 * np.cos(ph) + 0.08 * np.cos(2.0 * ph)
    return np.clip(v, 0.0, 1.0)


def pad_index_map(n: int, left: int, right: int, mode: str) -> np.ndarray:
    """Padded position -> source sample index (-1 = zero slot).

    signal.py:138-156 (np.pad 'reflect' mirrors without repeating the edge)
    and gradients.py:18-25 (the same map used to fold input gradients).
    """
    if left < 0 or right < 0:
        raise ValueError("pad amounts must be non-negative")
    idx = np.arange(n)
    if mode == "reflect":
        if left >= n or right >= n:
            raise ValueError("reflect padding must be shorter than the signal")
        return np.pad(idx, (left, right), mode="reflect")
    if mode == "constant_zero":
        return np.pad(idx, (left, right), constant_values=-1)
    raise ValueError(f"unknown pad mode {mode!r}")


def pad(x: np.ndarray, left: int, right: int, mode: str) -> np.ndarray:
    """signal.py:138-156 on the last axis (batched)."""
    m = pad_index_map(x.shape[-1], left, right, mode)
    out = x[..., np.maximum(m, 0)]
    if mode == "constant_zero":
        out = np.where(m >= 0, out, 0.0)
    return out


def strided_correlate(x: np.ndarray, bank: np.ndarray, stride: int) -> np.ndarray:
    """signal.py:159-183 -- out[r, t] = sum_m x[t*stride + m] * bank[r, m].

    Frames are materialised exactly as the reference does and multiplied with
    one DGEMM, so the oracle follows the reference's own arithmetic order.
    """
    bank = np.atleast_2d(np.asarray(bank))
    if np.iscomplexobj(bank):
        raise ValueError("kernels must be real")
    if bank.size == 0:
        raise ValueError("at least one non-empty kernel row is required")
    width = bank.shape[1]
    if width > x.shape[-1]:
        raise ValueError("kernel length exceeds signal length")
    if stride < 1:
        raise ValueError("stride must be >= 1")
    fr = np.ascontiguousarray(sliding_window_view(x, width)[::stride])
    return np.ascontiguousarray((fr @ bank.astype(np.float64).T).T)


def lowpass_taps(num_taps: int, cutoff: float, kind: str = "hamming") -> np.ndarray:
    """signal.py:186-211 -- windowed sinc, symmetrised, unit DC gain."""
    if num_taps < 3 or num_taps % 2 == 0:
        raise ValueError("num_taps must be an odd integer >= 3")
    if not 0.0 < cutoff < 1.0:
        raise ValueError("cutoff must lie in (0, 1)")
    c = (num_taps - 1) / 2.0
    h = cutoff * np.sinc(cutoff * (np.arange(num_taps) - c)) * window(kind, num_taps, False)
    h = 0.5 * (h + h[::-1])
    return h / h.sum()


def halve_rate(x: np.ndarray, taps: np.ndarray) -> np.ndarray:
    """signal.py:232-247 -- reflect pad (taps-1)/2, full-rate 'valid' FIR, keep [::2]."""
    if taps.size % 2 == 0:
        raise ValueError("odd-length filter required")
    if x.shape[-1] < taps.size:
        raise ValueError("signal shorter than filter")
    h = (taps.size - 1) // 2
    xp = pad(x, h, h, "reflect")
    return np.convolve(xp, taps, mode="valid")[::2]


# ----------------------------------------------------------------------------
# kernel banks                                                  (kernels.py)
# ----------------------------------------------------------------------------


def freq_ladder(kind: str, n_fft: int, sr: float, fmin: float = 50.0, fmax: float = 6000.0,
                n_bins: int | None = None) -> np.ndarray:
    """kernels.py:66-105 -- normalised frequencies (cycles per window)."""
    if n_bins is None:
        n_bins = n_fft // 2 + 1
    if not 1 <= n_bins <= n_fft // 2 + 1:
        raise ValueError("n_bins out of range")
    k = np.arange(n_bins, dtype=np.float64)
    if kind == "no":
        return k
    if not 0.0 < fmin < fmax or fmax > sr / 2.0:
        raise ValueError("bad fmin/fmax")
    start = fmin * n_fft / sr
    if kind == "linear":
        return (fmax - fmin) * n_fft / (n_bins * sr) * k + start
    if kind == "log":
        return start * (fmax / fmin) ** (k / n_bins)
    raise ValueError(f"unknown frequency scale {kind!r}")


def dft_bank(nf: np.ndarray, win: np.ndarray):
    """kernels.py:137-146 -- (cos*w, sin*w) rows; frame value is re - i*im."""
    n = win.size
    ph = 2.0 * np.pi * np.outer(nf, np.arange(n)) / n
    return np.cos(ph) * win, np.sin(ph) * win


_SL_F, _SL_M, _SL_STEP = 1000.0, 15.0, 27.0 / math.log(6.4)


def hz2mel(f, formula: str = "htk"):
    """kernels.py:158-171."""
    f = np.asarray(f, dtype=np.float64)
    if formula == "htk":
        return 2595.0 * np.log10(1.0 + f / 700.0)
    lin = 3.0 * f / 200.0
    return np.where(f < _SL_F, lin, _SL_M + _SL_STEP * np.log(np.maximum(f, _SL_F) / _SL_F))


def mel2hz(m, formula: str = "htk"):
    """kernels.py:174-183."""
    m = np.asarray(m, dtype=np.float64)
    if formula == "htk":
        return 700.0 * (10.0 ** (m / 2595.0) - 1.0)
    return np.where(m < _SL_M, 200.0 * m / 3.0,
                    _SL_F * np.exp(np.maximum(m - _SL_M, 0.0) / _SL_STEP))


def mel_bank(sr: float, n_fft: int, n_mels: int, fmin: float = 0.0, fmax: float | None = None,
             formula: str = "htk", norm: str = "none") -> np.ndarray:
    """kernels.py:214-254 -- triangles on n_mels+2 mel-spaced points."""
    if fmax is None:
        fmax = sr / 2.0
    pts = mel2hz(np.linspace(hz2mel(fmin, formula), hz2mel(fmax, formula), n_mels + 2), formula)
    fb = np.arange(n_fft // 2 + 1) * (sr / n_fft)
    w = np.zeros((n_mels, fb.size))
    for m in range(n_mels):
        lo, ce, hi = pts[m], pts[m + 1], pts[m + 2]
        tri = np.maximum(0.0, np.minimum((fb - lo) / (ce - lo), (hi - fb) / (hi - ce)))
        pk = tri.max()
        if pk == 0.0:
            pass
        elif norm == "none":
            tri = tri / pk
        else:
            tri = tri * (2.0 / (hi - lo))
        w[m] = tri
    return w


def cqt_quality(b: int) -> float:
    """kernels.py:261-265."""
    return 1.0 / (2.0 ** (1.0 / b) - 1.0)


@dataclass(frozen=True)
class CqtCfg:
    """kernels.py:275-321 (CqtConfig) -- fmax overrides n_bins."""

    sr: float
    fmin: float = 32.70
    n_bins: int = 84
    bins_per_octave: int = 12
    hop_length: int = 512
    window_kind: str = "hann"
    norm: int | None = 1
    fmax: float | None = None
    pad_mode: str = "reflect"
    early_downsample: bool = True
    downsample_taps: int = 255

    def __post_init__(self):
        if self.fmax is not None:
            object.__setattr__(self, "n_bins",
                               int(math.floor(self.bins_per_octave * math.log2(self.fmax / self.fmin))) + 1)
        top = self.fmin * 2.0 ** ((self.n_bins - 1) / self.bins_per_octave)
        if top >= self.sr / 2.0:
            raise ValueError("top bin reaches Nyquist")

    def freqs(self) -> np.ndarray:
        return self.fmin * 2.0 ** (np.arange(self.n_bins, dtype=np.float64) / self.bins_per_octave)


def cqt_time_bank(cfg: CqtCfg):
    """kernels.py:361-410 (domain='time') -- complex rows centred at width//2.

    Returns (kernels complex (n_bins, width), lengths)."""
    q = cqt_quality(cfg.bins_per_octave)
    f = cfg.freqs()
    lens = np.ceil(q * cfg.sr / f).astype(np.int64)
    width = int(lens[0]) + (int(lens[0]) & 1)
    k = np.zeros((cfg.n_bins, width), dtype=np.complex128)
    for r in range(cfg.n_bins):
        n_k = int(lens[r])
        v = np.exp(-2j * np.pi * (f[r] / cfg.sr) * np.arange(n_k)) * window(cfg.window_kind, n_k, True)
        if cfg.norm == 1:
            v = v / np.abs(v).sum()
        elif cfg.norm == 2:
            v = v / np.sqrt((np.abs(v) ** 2).sum())
        s = width // 2 - n_k // 2
        k[r, s:s + n_k] = v
    return k, lens


# ----------------------------------------------------------------------------
# transforms                                                 (transforms.py)
# ----------------------------------------------------------------------------


def _finish(re, im, output):
    """transforms.py:86-93."""
    if output == "complex":
        return re - 1j * im
    if output == "magnitude":
        return np.hypot(re, im)
    if output == "power":
        return re * re + im * im
    raise ValueError(output)


def _finish_complex(z, output):
    """transforms.py:96-103."""
    if output == "complex":
        return z
    if output == "magnitude":
        return np.abs(z)
    if output == "power":
        return z.real ** 2 + z.imag ** 2
    raise ValueError(output)


def stft_clip(x: np.ndarray, h_re: np.ndarray, h_im: np.ndarray, hop: int, center: bool = True,
              pad_mode: str = "reflect", output: str = "magnitude") -> np.ndarray:
    """transforms.py:130-144 -- centre pad n_fft//2, one DGEMM, finish."""
    n_fft = h_re.shape[1]
    if center:
        x = pad(x, n_fft // 2, n_fft // 2, pad_mode)
    fr = strided_correlate(x, np.vstack([h_re, h_im]), hop)
    nb = h_re.shape[0]
    return _finish(fr[:nb], fr[nb:], output)


def stft_bank(n_fft=2048, sr=44100.0, window_kind="hann", freq_scale="no", fmin=50.0, fmax=6000.0,
              freq_bins=None):
    """transforms.py:118-128 -- the Stft constructor's bank."""
    nf = freq_ladder(freq_scale, n_fft, sr, fmin, fmax, freq_bins)
    return dft_bank(nf, window(window_kind, n_fft, True))


def mel_clip(x, h_re, h_im, W, hop, power=1.0, center=True, pad_mode="reflect"):
    """transforms.py:164-172 -- W @ |STFT|**power."""
    mag = stft_clip(x, h_re, h_im, hop, center, pad_mode, "magnitude")
    if power != 1.0:
        mag = mag ** power
    return W @ mag


def cqt1992v2_clip(x, kern: np.ndarray, hop: int, pad_mode="reflect", output="magnitude"):
    """transforms.py:175-186 + 201-208 -- centred complex conv with the long bank."""
    width = kern.shape[1]
    xp = pad(x, width // 2, width // 2, pad_mode)
    fr = strided_correlate(xp, np.vstack([kern.real, kern.imag]), hop)
    r = kern.shape[0]
    return _finish_complex(fr[:r] + 1j * fr[r:], output)


@dataclass
class Cqt2010Plan:
    """transforms.py:249-285 -- octave recursion bookkeeping."""

    n_octaves: int
    n_filters: int
    first_bin: int
    early_stages: int
    kernel_hop: int
    kernel_sr: float
    top_kernels: np.ndarray
    taps: np.ndarray


def cqt2010_plan(cfg: CqtCfg) -> Cqt2010Plan:
    b = cfg.bins_per_octave
    n_oct = math.ceil(cfg.n_bins / b)
    div = 2 ** (n_oct - 1)
    if cfg.hop_length % div != 0:
        raise ValueError(f"hop_length must be divisible by 2**(n_octaves - 1) = {div}")
    n_filt = min(b, cfg.n_bins)
    first = cfg.n_bins - n_filt
    f_top = cfg.fmin * 2.0 ** ((cfg.n_bins - 1) / b)
    m = 0
    if cfg.early_downsample:
        lim = cfg.sr / (2.0 * 1.3 * f_top)
        if lim > 1.0:
            m = int(math.floor(math.log2(lim)))
        while m > 0 and cfg.hop_length % (2 ** (m + n_oct - 1)) != 0:
            m -= 1
    ksr = cfg.sr / 2 ** m
    khop = cfg.hop_length // 2 ** m
    top = CqtCfg(sr=ksr, fmin=cfg.fmin * 2.0 ** (first / b), n_bins=n_filt, bins_per_octave=b,
                 hop_length=max(1, khop // div), window_kind=cfg.window_kind, norm=cfg.norm,
                 pad_mode=cfg.pad_mode, early_downsample=False)
    kern, _ = cqt_time_bank(top)
    return Cqt2010Plan(n_oct, n_filt, first, m, khop, ksr, kern,
                       lowpass_taps(cfg.downsample_taps, 0.5, "hamming"))


def cqt2010v2_clip(x, cfg: CqtCfg, plan: Cqt2010Plan | None = None, output="magnitude"):
    """transforms.py:290-313 + 319-323 -- early halvings, then per octave:
    halve (alpha>0), centred complex conv at hop kernel_hop>>alpha, trim to the
    shortest octave, scatter rows to first_bin + skip + j - alpha*b."""
    p = plan or cqt2010_plan(cfg)
    cur = x
    for _ in range(p.early_stages):
        cur = halve_rate(cur, p.taps)
    b = cfg.bins_per_octave
    octs = []
    for a in range(p.n_octaves):
        if a > 0:
            cur = halve_rate(cur, p.taps)
        fr = cqt1992v2_clip(cur, p.top_kernels, p.kernel_hop >> a, cfg.pad_mode, "complex")
        skip = max(0, a * b - p.first_bin)
        octs.append((a, skip, fr[skip:]))
    nfr = min(f.shape[1] for _, _, f in octs)
    out = np.zeros((cfg.n_bins, nfr), dtype=np.complex128)
    for a, skip, fr in octs:
        for j in range(fr.shape[0]):
            out[p.first_bin + skip + j - a * b] = fr[j, :nfr]
    return _finish_complex(out, output)


def cqt_freq_bank(cfg: CqtCfg):
    """kernels.py:361-410 (domain='frequency') -- kernels centred in rows of
    fft_len = next power of two >= N_0, and their spectra with the reversed
    index sign: freq_kernels = conj(fft(conj(time_kernels))).  Returns
    (freq_kernels, fft_len)."""
    q = cqt_quality(cfg.bins_per_octave)
    f = cfg.freqs()
    lens = np.ceil(q * cfg.sr / f).astype(np.int64)
    n = 1
    while n < int(lens[0]):
        n *= 2
    k = np.zeros((cfg.n_bins, n), dtype=np.complex128)
    for r in range(cfg.n_bins):
        n_k = int(lens[r])
        v = np.exp(-2j * np.pi * (f[r] / cfg.sr) * np.arange(n_k)) * window(cfg.window_kind, n_k, True)
        if cfg.norm == 1:
            v = v / np.abs(v).sum()
        elif cfg.norm == 2:
            v = v / np.sqrt((np.abs(v) ** 2).sum())
        s0 = n // 2 - n_k // 2
        k[r, s0:s0 + n_k] = v
    return np.conj(np.fft.fft(np.conj(k), axis=1)), n


def _freq_domain_frames(x, freq_kernels, n, hop, pad_mode):
    """transforms.py:229-235 / 333-337 -- centre pad n//2, full-spectrum DFT of
    every frame (the reference's rectangular DFT bank conv; here np.fft of the
    same frames), then the spectral product with the kernels / n."""
    xp = pad(x, n // 2, n // 2, pad_mode)
    if n > xp.size:
        raise ValueError("signal shorter than kernel")
    fr = sliding_window_view(xp, n)[::hop]
    spectra = np.fft.fft(fr, axis=1)  # sum_m x[m] e^{-2 pi i k m / n} = frames[:n] - 1j * frames[n:]
    return (spectra @ freq_kernels.T).T / n


def cqt1992_clip(x, cfg: CqtCfg, output="magnitude"):
    """transforms.py:211-238 (Cqt1992) -- constant-Q through the frequency domain."""
    fk, n = cqt_freq_bank(cfg)
    return _finish_complex(_freq_domain_frames(x, fk, n, cfg.hop_length, cfg.pad_mode), output)


def cqt2010_clip(x, cfg: CqtCfg, plan: Cqt2010Plan | None = None, output="magnitude"):
    """transforms.py:326-337 (Cqt2010) -- the octave recursion of cqt2010v2_clip
    with each octave's conv done through the frequency domain (top-octave bank,
    fft_len of its longest kernel)."""
    p = plan or cqt2010_plan(cfg)
    b = cfg.bins_per_octave
    top = CqtCfg(sr=p.kernel_sr, fmin=cfg.fmin * 2.0 ** (p.first_bin / b), n_bins=p.n_filters, bins_per_octave=b,
                 hop_length=max(1, p.kernel_hop // 2 ** (p.n_octaves - 1)), window_kind=cfg.window_kind,
                 norm=cfg.norm, pad_mode=cfg.pad_mode, early_downsample=False)
    fk, n = cqt_freq_bank(top)
    cur = x
    for _ in range(p.early_stages):
        cur = halve_rate(cur, p.taps)
    octs = []
    for a in range(p.n_octaves):
        if a > 0:
            cur = halve_rate(cur, p.taps)
        fr = _freq_domain_frames(cur, fk, n, p.kernel_hop >> a, cfg.pad_mode)
        skip = max(0, a * b - p.first_bin)
        octs.append((a, skip, fr[skip:]))
    nfr = min(f.shape[1] for _, _, f in octs)
    out = np.zeros((cfg.n_bins, nfr), dtype=np.complex128)
    for a, skip, fr in octs:
        for j in range(fr.shape[0]):
            out[p.first_bin + skip + j - a * b] = fr[j, :nfr]
    return _finish_complex(out, output)


def map_clips(fn, clips: np.ndarray, threads: int | None = None) -> np.ndarray:
    """transforms.py:370-388 (batch_transform) -- ordered map over clips with
    an optional thread pool; results identical to the sequential map."""
    if threads is None:
        threads = int(os.environ.get("SPECTRO_THREADS", "1"))
    if threads <= 1:
        return np.stack([fn(c) for c in clips])
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return np.stack(list(ex.map(fn, clips)))


# ----------------------------------------------------------------------------
# trainable layers                                           (gradients.py)
# ----------------------------------------------------------------------------


def _frames(x, width, hop, center, pad_mode):
    """gradients.py:49-59."""
    if center:
        x = pad(x, width // 2, width // 2, pad_mode)
    if x.size < width:
        raise ValueError("signal too short")
    return np.ascontiguousarray(sliding_window_view(x, width)[::hop])


def smooth_mag_forward(x, h_re, h_im, hop, eps=1e-12, center=True, pad_mode="reflect"):
    """gradients.py:61-67 -- frames, re, im, S = sqrt(re^2 + im^2 + eps) (bins x frames)."""
    fr = _frames(x, h_re.shape[1], hop, center, pad_mode)
    re = fr @ h_re.T
    im = fr @ h_im.T
    return fr, re.T, im.T, np.sqrt(re * re + im * im + eps).T


def mel_layer_forward(x, W, h_re, h_im, hop, eps=1e-12, center=True, pad_mode="reflect"):
    """gradients.py:69-80 -- W @ smoothed STFT magnitude (fixed STFT stage)."""
    return W @ smooth_mag_forward(x, h_re, h_im, hop, eps, center, pad_mode)[3]


def conv_layer_vjp(x, h_re, h_im, hop, g, eps=1e-12, center=True, pad_mode="reflect",
                   with_input_grad=False):
    """gradients.py:103-149 -- dh_re = (g*re/S) @ frames, dh_im likewise;
    optional dx = overlap-add of coef^T @ h folded through the pad map."""
    fr, re, im, S = smooth_mag_forward(x, h_re, h_im, hop, eps, center, pad_mode)
    if g.shape != S.shape:
        raise ValueError("upstream_grad shape mismatch")
    cre, cim = g * (re / S), g * (im / S)
    grads = {"h_re": cre @ fr, "h_im": cim @ fr}
    if not with_input_grad:
        return grads
    width = h_re.shape[1]
    fg = cre.T @ h_re + cim.T @ h_im
    p = width // 2 if center else 0
    gp = np.zeros(x.size + 2 * p)
    pos = (np.arange(fg.shape[0]) * hop)[:, None] + np.arange(width)[None, :]
    np.add.at(gp, pos.ravel(), fg.ravel())
    gx = np.zeros(x.size)
    if center:
        m = pad_index_map(x.size, p, p, pad_mode)
        keep = m >= 0
        np.add.at(gx, m[keep], gp[keep])
    else:
        gx += gp
    return grads, gx


def mel_layer_vjp(x, W, h_re, h_im, hop, g, eps=1e-12, center=True, pad_mode="reflect"):
    """gradients.py:118-124 -- dW = g @ S^T."""
    S = smooth_mag_forward(x, h_re, h_im, hop, eps, center, pad_mode)[3]
    return {"weights": g @ S.T}


def peak_err(got, ref) -> float:
    """Peak-normalised max error, the metric every reference test uses
    (tests/test_transforms.py:60, tests/test_acceptance.py:97)."""
    ref = np.asarray(ref)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(np.asarray(got) - ref)) / (den if den > 0 else 1.0))
