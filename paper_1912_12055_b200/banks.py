"""Init-time kernel banks (host, float64), built once per transform.

These restate the reference's bank factories (kernels.py) so transforms own
their banks exactly as `spectro` does; the banks are then uploaded once and
packed into the sm_100a GEMM operand layout on the device.
Citations are relative to /root/reference/pkg/src/spectro/.
"""

from __future__ import annotations

import math
import warnings

import numpy as np

WINDOW_KINDS = ("hann", "hamming", "blackman", "rectangular")
FREQ_SCALES = ("no", "linear", "log")


def make_window(kind: str, n: int, periodic: bool = True) -> np.ndarray:
    """signal.py:106-135: cosine-sum windows clipped to [0, 1]."""
    if n < 1:
        raise ValueError(f"window length must be >= 1, got {n}")
    if kind not in WINDOW_KINDS:
        raise ValueError(f"unknown window kind {kind!r}; expected one of {WINDOW_KINDS}")
    if kind == "rectangular":
        return np.ones(n)
    denom = n if periodic else n - 1
    if denom == 0:
        return np.ones(1)
    a = {"hann": (0.5, 0.5, 0.0), "hamming": (0.54, 0.46, 0.0), "blackman": (0.42, 0.5, 0.08)}[kind]
    t = 2.0 * np.pi * np.arange(n) / denom
    v = a[0] - a[1] * np.cos(t)
    if a[2]:
        v = v + a[2] * np.cos(2.0 * t)
    return np.clip(v, 0.0, 1.0)


def frequency_scale(kind: str, n_fft: int, sr: float, fmin: float, fmax: float, n_bins: int | None):
    """kernels.py:66-105 -> (normalised frequencies, bin_freqs_hz)."""
    if kind not in FREQ_SCALES:
        raise ValueError(f"unknown frequency scale {kind!r}; expected one of {FREQ_SCALES}")
    if n_fft < 1:
        raise ValueError("n_fft must be >= 1")
    if sr <= 0:
        raise ValueError("sample_rate must be positive")
    n_bins = n_fft // 2 + 1 if n_bins is None else n_bins
    if not 1 <= n_bins <= n_fft // 2 + 1:
        raise ValueError(f"n_bins must lie in [1, n_fft/2 + 1], got {n_bins}")
    k = np.arange(n_bins, dtype=np.float64)
    if kind == "no":
        nf = k
    else:
        if not 0.0 < fmin < fmax:
            raise ValueError(f"need 0 < fmin < fmax, got fmin={fmin}, fmax={fmax}")
        if fmax > sr / 2.0:
            raise ValueError(f"fmax={fmax} exceeds the Nyquist frequency {sr / 2.0}")
        k0 = fmin * n_fft / sr
        nf = (k0 + (fmax - fmin) * n_fft / (n_bins * sr) * k) if kind == "linear" else k0 * (fmax / fmin) ** (k / n_bins)
    return nf, nf * (sr / n_fft)


def dft_kernels(norm_freqs: np.ndarray, window: np.ndarray):
    """kernels.py:137-146: rows cos(2 pi f n / N) w[n] and sin(...) w[n]."""
    n = window.size
    phase = (2.0 * np.pi / n) * np.outer(norm_freqs, np.arange(n))
    return np.cos(phase) * window, np.sin(phase) * window


def hz_to_mel(f, formula="htk"):
    """kernels.py:158-171."""
    f = np.asarray(f, dtype=np.float64)
    if np.any(f < 0):
        raise ValueError("frequencies must be non-negative")
    if formula == "htk":
        return 2595.0 * np.log10(1.0 + f / 700.0)
    if formula == "slaney":
        logstep = 27.0 / math.log(6.4)
        return np.where(f < 1000.0, 3.0 * f / 200.0, 15.0 + logstep * np.log(np.maximum(f, 1000.0) / 1000.0))
    raise ValueError(f"unknown mel formula {formula!r}")


def mel_to_hz(m, formula="htk"):
    """kernels.py:174-183."""
    m = np.asarray(m, dtype=np.float64)
    if formula == "htk":
        return 700.0 * (10.0 ** (m / 2595.0) - 1.0)
    if formula == "slaney":
        logstep = 27.0 / math.log(6.4)
        return np.where(m < 15.0, 200.0 * m / 3.0, 1000.0 * np.exp(np.maximum(m - 15.0, 0.0) / logstep))
    raise ValueError(f"unknown mel formula {formula!r}")


def mel_filter_bank(sr: float, n_fft: int, n_mels: int, fmin: float = 0.0, fmax: float | None = None,
                    formula: str = "htk", norm: str = "none"):
    """kernels.py:214-254 -> (weights (n_mels, n_fft//2+1), centre freqs)."""
    fmax = sr / 2.0 if fmax is None else fmax
    if n_mels < 1:
        raise ValueError("n_mels must be >= 1")
    if not 0.0 <= fmin < fmax:
        raise ValueError(f"need 0 <= fmin < fmax, got fmin={fmin}, fmax={fmax}")
    if fmax > sr / 2.0:
        raise ValueError(f"fmax={fmax} exceeds the Nyquist frequency {sr / 2.0}")
    if norm not in ("none", "area"):
        raise ValueError(f"unknown norm {norm!r}; expected 'none' or 'area'")
    hz = mel_to_hz(np.linspace(hz_to_mel(fmin, formula), hz_to_mel(fmax, formula), n_mels + 2), formula)
    fb = np.arange(n_fft // 2 + 1) * (sr / n_fft)
    left, centre, right = hz[:-2, None], hz[1:-1, None], hz[2:, None]
    tri = np.maximum(0.0, np.minimum((fb - left) / (centre - left), (right - fb) / (right - centre)))
    peak = tri.max(axis=1, keepdims=True)
    if (peak[:, 0] == 0).any():  # kernels.py: an n_fft too small for n_mels leaves empty rows
        warnings.warn(f"{int((peak[:, 0] == 0).sum())} of {n_mels} mel filters are empty; "
                      "increase n_fft or reduce n_mels", UserWarning, stacklevel=2)
    if norm == "none":
        w = np.where(peak > 0, tri / np.where(peak > 0, peak, 1.0), tri)
    else:
        w = tri * (2.0 / (right - left))
    return w, hz[1:-1]


def cqt_q(bins_per_octave: int) -> float:
    """kernels.py:261-265."""
    if bins_per_octave < 1:
        raise ValueError("bins_per_octave must be >= 1")
    return 1.0 / (2.0 ** (1.0 / bins_per_octave) - 1.0)


def cqt_time_kernels(sr: float, freqs: np.ndarray, bins_per_octave: int, window_kind: str, norm):
    """kernels.py:361-402 (time domain): complex rows exp(-2 pi i f_k n / sr) * w_k,
    normalised, centred at column width//2 of an even-width row.
    Returns (kernels complex128 (n_bins, width), lengths int64)."""
    q = cqt_q(bins_per_octave)
    lengths = np.ceil(q * sr / freqs).astype(np.int64)
    width = int(lengths[0]) + (int(lengths[0]) & 1)
    out = np.zeros((freqs.size, width), dtype=np.complex128)
    for r, (f, n_k) in enumerate(zip(freqs, lengths)):
        n = np.arange(int(n_k))
        v = np.exp(-2j * np.pi * (f / sr) * n) * make_window(window_kind, int(n_k), True)
        if norm == 1:
            v /= np.abs(v).sum()
        elif norm == 2:
            v /= np.sqrt((np.abs(v) ** 2).sum())
        s = width // 2 - int(n_k) // 2
        out[r, s:s + int(n_k)] = v
    return out, lengths


def lowpass_fir(num_taps: int, cutoff: float, window_kind: str = "hamming") -> np.ndarray:
    """signal.py:186-211: symmetric windowed sinc with unit DC gain."""
    if num_taps < 3 or num_taps % 2 == 0:
        raise ValueError(f"num_taps must be an odd integer >= 3, got {num_taps}")
    if not 0.0 < cutoff < 1.0:
        raise ValueError(f"cutoff must lie in (0, 1), got {cutoff}")
    c = (num_taps - 1) / 2.0
    h = cutoff * np.sinc(cutoff * (np.arange(num_taps) - c)) * make_window(window_kind, num_taps, periodic=False)
    h = 0.5 * (h + h[::-1])
    return h / h.sum()


def mel_bands(weights: np.ndarray, n_chunks: int, chunk: int = 32) -> np.ndarray:
    """[lo, hi) mel rows with a non-zero weight in each `chunk`-bin slice: the
    fused epilogue only visits those rows (the default bank is 1.5 % dense)."""
    nz = weights != 0
    band = np.zeros((n_chunks, 2), dtype=np.int32)
    for c in range(n_chunks):
        rows = np.nonzero(nz[:, c * chunk:(c + 1) * chunk].any(axis=1))[0]
        if rows.size:
            band[c] = (rows[0], rows[-1] + 1)
    return band
