"""`spectro`-compatible transforms on the sm_100a kernels.

Same class / function names, argument meanings and error behaviour as the
reference's transform layer (/root/reference/pkg/src/spectro/transforms.py)
so callers and the reference's own tests can switch backends; the work runs
batched on the GPU through the C ABI (engine.py).  Differences by design:
`Signal.samples` and `Spectrogram.data` are CUDA tensors (float32, complex64
for complex output), and `batch_transform` runs a whole batch in one launch
instead of a thread pool (still order-preserving and identical to the
sequential map).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import banks
from .engine import CqtLongEngine, Cqt2010Engine, DftEngine, _require_cuda

OUTPUT_KINDS = ("complex", "magnitude", "power")


@dataclass(frozen=True)
class Signal:
    """signal.py:22-49 -- a mono float sample sequence and its rate (finite, sr > 0)."""

    samples: torch.Tensor
    sample_rate: float
    device: str = field(default="cuda", compare=False)

    def __post_init__(self):
        s = self.samples
        s = s.detach() if torch.is_tensor(s) else torch.as_tensor(np.asarray(s, dtype=np.float32))
        s = s.to(_require_cuda(self.device), torch.float32)
        if s.dim() != 1:
            raise ValueError(f"samples must be 1-D, got shape {tuple(s.shape)}")
        if not bool(torch.isfinite(s).all()):
            raise ValueError("samples must be finite (no NaN/Inf)")
        if not self.sample_rate > 0:
            raise ValueError(f"sample_rate must be positive, got {self.sample_rate}")
        object.__setattr__(self, "samples", s)
        object.__setattr__(self, "sample_rate", float(self.sample_rate))

    def __len__(self):
        return int(self.samples.shape[0])

    @property
    def duration(self) -> float:
        return len(self) / self.sample_rate


@dataclass(frozen=True)
class Spectrogram:
    """transforms.py:24-47 -- bins x frames plus the metadata to interpret it."""

    data: torch.Tensor
    bin_freqs_hz: np.ndarray | None
    hop: int
    sample_rate: float
    kind: str

    def __post_init__(self):
        if self.kind not in OUTPUT_KINDS:
            raise ValueError(f"kind must be one of {OUTPUT_KINDS}, got {self.kind!r}")

    @property
    def n_bins(self):
        return int(self.data.shape[0])

    @property
    def n_frames(self):
        return int(self.data.shape[1])


# ------------------------------------------------------------- signal primitives
# signal.py's building blocks on the device (the transforms below fuse them
# into their own kernels; these serve direct callers and the primitives' KATs).

PAD_MODES = {"reflect": 0, "constant_zero": 1}


@dataclass(frozen=True)
class FrameMatrix:
    """signal.py:91-103 -- kernel responses per frame: values (n_kernels, n_frames)."""

    values: torch.Tensor
    hop: int = 1

    @property
    def n_frames(self):
        return int(self.values.shape[1])


@dataclass(frozen=True)
class FirFilter:
    """signal.py:76-88 -- FIR taps (float64, host) and their normalised cutoff."""

    taps: np.ndarray
    normalized_cutoff: float


def make_window(kind: str, n: int, periodic: bool = True) -> np.ndarray:
    """signal.py:106-135 (host, init-time)."""
    return banks.make_window(kind, n, periodic)


def design_lowpass_fir(num_taps: int, cutoff: float, window_kind: str = "hamming") -> FirFilter:
    """signal.py:186-211 (host, init-time)."""
    return FirFilter(banks.lowpass_fir(num_taps, cutoff, window_kind), float(cutoff))


def pad_signal(x: Signal, mode: str, left: int, right: int) -> Signal:
    """signal.py:138-156 on the device (nnab_pad_signal), bit-exact."""
    from . import _lib as L
    if left < 0 or right < 0:
        raise ValueError("pad amounts must be non-negative")
    if mode not in PAD_MODES:
        raise ValueError(f"unknown pad mode {mode!r}")
    n = len(x)
    if mode == "reflect" and (left >= n or right >= n):
        raise ValueError(f"reflect padding ({left}, {right}) must be shorter than the signal (len {n})")
    y = torch.empty(n + left + right, dtype=torch.float32, device=x.samples.device)
    L.check(L.load().nnab_pad_signal(x.samples.data_ptr(), 1, n, int(left), int(right), PAD_MODES[mode],
                                     y.data_ptr(), L.stream_handle(y.device)), "pad_signal")
    return Signal(y, x.sample_rate, device=str(y.device))


def conv1d_strided(x: Signal, kernels, stride: int, precision: str = "fp32") -> FrameMatrix:
    """signal.py:159-183: out[r, t] = sum_m x[t*stride + m] * kernels[r, m] (no
    padding, cross-correlation), on the tcgen05 GEMM (a real bank as the
    cosine rows of a DFT-type bank with zero sine rows, complex output).
    precision "fp32" (3xTF32, default: FP32-accurate) or "tf32"."""
    k = kernels.detach().cpu().numpy() if torch.is_tensor(kernels) else np.asarray(kernels)
    k = np.atleast_2d(k)
    if np.iscomplexobj(k):
        raise ValueError("kernels must be real; run real and imaginary parts separately")
    if k.size == 0:
        raise ValueError("at least one non-empty kernel row is required")
    m = k.shape[1]
    if m > len(x):
        raise ValueError(f"kernel length {m} exceeds signal length {len(x)}; pad the signal first")
    if stride < 1:
        raise ValueError(f"stride must be >= 1, got {stride}")
    k32 = k.astype(np.float32)
    eng = DftEngine(k32, np.zeros_like(k32), int(stride), center=False, precision=precision,
                    device=x.samples.device, allow_fold=False)
    out = eng.forward(x.samples[None], "complex")[0]  # re - i*im with zero sine rows: re
    return FrameMatrix(out.real.contiguous(), hop=int(stride))


def downsample2(x: Signal, f: FirFilter) -> Signal:
    """signal.py:232-247 on the device (nnab_downsample2): reflect pad, FIR,
    keep every second sample; FP32 accumulation."""
    from . import _lib as L
    taps = np.asarray(f.taps if isinstance(f, FirFilter) else f, dtype=np.float64)
    if taps.size % 2 == 0:
        raise ValueError("downsample2 requires an odd-length (center-tap) filter")
    if len(x) < taps.size:
        raise ValueError(f"signal (len {len(x)}) shorter than filter (len {taps.size})")
    dev = x.samples.device
    t = torch.as_tensor(taps, dtype=torch.float32, device=dev)
    y = torch.empty((len(x) + 1) // 2, dtype=torch.float32, device=dev)
    L.check(L.load().nnab_downsample2(x.samples.data_ptr(), 1, len(x), t.data_ptr(), int(taps.size), y.data_ptr(),
                                      L.stream_handle(dev)), "downsample2")
    return Signal(y, x.sample_rate / 2.0, device=str(dev))


@dataclass(frozen=True)
class StftParams:
    """transforms.py:50-65."""

    n_fft: int = 2048
    freq_bins: int | None = None
    hop_length: int = 512
    window: str = "hann"
    freq_scale: str = "no"
    center: bool = True
    pad_mode: str = "reflect"
    fmin: float = 50.0
    fmax: float = 6000.0
    output: str = "magnitude"


@dataclass(frozen=True)
class MelParams:
    """transforms.py:68-83 (default: slaney, peak-normalised, magnitude)."""

    sr: float | None = None
    n_fft: int = 2048
    n_mels: int = 128
    hop_length: int = 512
    window: str = "hann"
    center: bool = True
    pad_mode: str = "reflect"
    htk: bool = False
    fmin: float = 0.0
    fmax: float | None = None
    norm: str = "none"
    power: float = 1.0


@dataclass(frozen=True)
class CqtConfig:
    """kernels.py:275-321 -- fmax overrides n_bins; the top bin must stay below Nyquist."""

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
        if self.sr <= 0:
            raise ValueError("sr must be positive")
        if self.fmin <= 0:
            raise ValueError("fmin must be positive")
        if self.bins_per_octave < 1:
            raise ValueError("bins_per_octave must be >= 1")
        if self.hop_length < 1:
            raise ValueError("hop_length must be >= 1")
        if self.norm not in (1, 2, None):
            raise ValueError("norm must be 1, 2, or None")
        if self.fmax is not None:
            object.__setattr__(self, "n_bins",
                               int(math.floor(self.bins_per_octave * math.log2(self.fmax / self.fmin))) + 1)
        if self.n_bins < 1:
            raise ValueError("n_bins must be >= 1")
        top = self.fmin * 2.0 ** ((self.n_bins - 1) / self.bins_per_octave)
        if top >= self.sr / 2.0:
            raise ValueError(f"top bin frequency {top:.2f} Hz reaches the Nyquist frequency "
                             f"{self.sr / 2.0:.2f} Hz; reduce n_bins or fmax")

    @property
    def bin_freqs_hz(self) -> np.ndarray:
        return self.fmin * 2.0 ** (np.arange(self.n_bins, dtype=np.float64) / self.bins_per_octave)


def _check_output(output: str) -> str:
    if output not in OUTPUT_KINDS:
        raise ValueError(f"output must be one of {OUTPUT_KINDS}, got {output!r}")
    return output


class _Batched:
    """Shared helpers: one clip via the batched path; batch of clips in one launch."""

    sample_rate: float

    def _check_signal(self, x: Signal):
        if x.sample_rate != self.sample_rate:
            raise ValueError(f"signal rate {x.sample_rate} != transform rate {self.sample_rate}")
        if len(x) < 1:
            raise ValueError("signal must be non-empty")

    def __call__(self, x: Signal, *a, **kw) -> Spectrogram:
        self._check_signal(x)
        data, meta = self.batch(x.samples[None], *a, **kw)
        return Spectrogram(data=data[0], **meta)


class Stft(_Batched):
    """transforms.py:110-144 -- precomputed cos/sin kernels, tcgen05 GEMM on device."""

    def __init__(self, params: StftParams, sample_rate: float, precision: str = "tf32", device="cuda"):
        if params.output not in OUTPUT_KINDS:
            raise ValueError(f"output must be one of {OUTPUT_KINDS}")
        self.params = params
        self.sample_rate = float(sample_rate)
        nf, self.bin_freqs_hz = banks.frequency_scale(params.freq_scale, params.n_fft, sample_rate, params.fmin,
                                                      params.fmax, params.freq_bins)
        self.h_re, self.h_im = banks.dft_kernels(nf, banks.make_window(params.window, params.n_fft, True))
        self.engine = DftEngine(self.h_re, self.h_im, params.hop_length, params.center, params.pad_mode,
                                precision=precision, device=device)

    def batch(self, x: torch.Tensor, output: str | None = None):
        """(B, L) float32 CUDA tensor -> ((B, F, T) tensor, Spectrogram metadata)."""
        out = _check_output(output if output is not None else self.params.output)
        if x.shape[-1] < 1:
            raise ValueError("signal must be non-empty")
        data = self.engine.forward(x, out)
        return data, dict(bin_freqs_hz=self.bin_freqs_hz, hop=self.params.hop_length,
                          sample_rate=self.sample_rate, kind=out)


class MelSpec(_Batched):
    """transforms.py:147-172 -- W @ |STFT|**power with the projection fused
    into the STFT GEMM epilogue."""

    def __init__(self, params: MelParams, sample_rate: float, precision: str = "tf32", device="cuda"):
        if params.sr is not None and params.sr != sample_rate:
            raise ValueError(f"params.sr {params.sr} != sample_rate {sample_rate}")
        self.params = params
        self.sample_rate = float(sample_rate)
        nf, _ = banks.frequency_scale("no", params.n_fft, sample_rate, 50.0, 6000.0, None)
        h_re, h_im = banks.dft_kernels(nf, banks.make_window(params.window, params.n_fft, True))
        self.weights, self.mel_center_freqs_hz = banks.mel_filter_bank(
            sample_rate, params.n_fft, params.n_mels, fmin=params.fmin, fmax=params.fmax,
            formula="htk" if params.htk else "slaney", norm=params.norm)
        self.engine = DftEngine(h_re, h_im, params.hop_length, params.center, params.pad_mode,
                                precision=precision, device=device)
        self.engine.set_mel(self.weights, power=params.power)

    def batch(self, x: torch.Tensor):
        data = self.engine.forward(x, "mel")
        return data, dict(bin_freqs_hz=self.mel_center_freqs_hz, hop=self.params.hop_length,
                          sample_rate=self.sample_rate, kind="magnitude" if self.params.power == 1.0 else "power")


class Cqt1992v2(_Batched):
    """transforms.py:194-208 -- long time-domain complex bank, scheduled tcgen05 GEMM."""

    def __init__(self, cfg: CqtConfig, precision: str = "tf32", device="cuda"):
        self.cfg = cfg
        self.sample_rate = float(cfg.sr)
        self.kernels, self.lengths = banks.cqt_time_kernels(cfg.sr, cfg.bin_freqs_hz, cfg.bins_per_octave,
                                                            cfg.window_kind, cfg.norm)
        self.bin_freqs_hz = cfg.bin_freqs_hz
        self.engine = CqtLongEngine(self.kernels, cfg.hop_length, cfg.pad_mode, precision=precision, device=device)

    def _check_signal(self, x: Signal):
        if x.sample_rate != self.cfg.sr:
            raise ValueError(f"signal rate {x.sample_rate} != configured rate {self.cfg.sr}")

    def batch(self, x: torch.Tensor, output: str = "magnitude"):
        out = _check_output(output)
        data = self.engine.forward(x, out)
        return data, dict(bin_freqs_hz=self.bin_freqs_hz, hop=self.cfg.hop_length, sample_rate=self.cfg.sr,
                          kind=out)


def cqt2010_plan(cfg: CqtConfig) -> dict:
    """transforms.py:249-285 -- octave count, hop divisibility, early halvings,
    top-octave bank and the anti-alias FIR."""
    b = cfg.bins_per_octave
    n_oct = math.ceil(cfg.n_bins / b)
    divisor = 2 ** (n_oct - 1)
    if cfg.hop_length % divisor != 0:
        raise ValueError(f"hop_length must be divisible by 2**(n_octaves - 1) = {divisor}, got {cfg.hop_length}")
    n_filt = min(b, cfg.n_bins)
    first_bin = cfg.n_bins - n_filt
    f_top = cfg.fmin * 2.0 ** ((cfg.n_bins - 1) / b)
    m = 0
    if cfg.early_downsample:
        limit = cfg.sr / (2.0 * 1.3 * f_top)
        if limit > 1.0:
            m = int(math.floor(math.log2(limit)))
        while m > 0 and cfg.hop_length % (2 ** (m + n_oct - 1)) != 0:
            m -= 1
    kernel_sr = cfg.sr / 2 ** m
    kernel_hop = cfg.hop_length // 2 ** m
    top = CqtConfig(sr=kernel_sr, fmin=cfg.fmin * 2.0 ** (first_bin / b), n_bins=n_filt, bins_per_octave=b,
                    hop_length=max(1, kernel_hop // divisor), window_kind=cfg.window_kind, norm=cfg.norm,
                    pad_mode=cfg.pad_mode, early_downsample=False)
    top_k, _ = banks.cqt_time_kernels(top.sr, top.bin_freqs_hz, b, cfg.window_kind, cfg.norm)
    return {"n_octaves": n_oct, "n_filters": n_filt, "first_bin": first_bin, "early_stages": m,
            "kernel_sr": kernel_sr, "kernel_hop": kernel_hop, "top_kernels": top_k,
            "taps": banks.lowpass_fir(cfg.downsample_taps, 0.5, "hamming")}


class Cqt2010v2(_Batched):
    """transforms.py:241-323 -- octave recursion run entirely on the device."""

    def __init__(self, cfg: CqtConfig, device="cuda"):
        self.cfg = cfg
        self.sample_rate = float(cfg.sr)
        p = cqt2010_plan(cfg)
        self.n_octaves, self.early_stages = p["n_octaves"], p["early_stages"]
        self.kernel_hop, self.first_bin = p["kernel_hop"], p["first_bin"]
        self.engine = Cqt2010Engine(p["taps"], p["top_kernels"], p["early_stages"], p["n_octaves"],
                                    p["kernel_hop"], p["first_bin"], cfg.bins_per_octave, cfg.n_bins, cfg.pad_mode,
                                    device=device)

    def _check_signal(self, x: Signal):
        if x.sample_rate != self.cfg.sr:
            raise ValueError(f"signal rate {x.sample_rate} != configured rate {self.cfg.sr}")

    def batch(self, x: torch.Tensor, output: str = "magnitude"):
        out = _check_output(output)
        data = self.engine.forward(x, out)
        return data, dict(bin_freqs_hz=self.cfg.bin_freqs_hz, hop=self.cfg.hop_length, sample_rate=self.cfg.sr,
                          kind=out)


def _next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p *= 2
    return p


class Cqt1992(Cqt1992v2):
    """transforms.py:211-238 -- constant-Q through the frequency domain: centre
    pad fft_len // 2, full-spectrum DFT of every frame, product with the
    kernels' spectra / fft_len.  By the power theorem (kernels.py:403-407) that
    is exactly the centred time-domain correlation with the same kernels, which
    is what runs here (the reference documents the equivalence:
    tests/test_acceptance.py:116-126); only the reference's own constraints of
    the frequency route (its fft_len // 2 reflect pad) are checked on top."""

    def __init__(self, cfg: CqtConfig, precision: str = "tf32", device="cuda"):
        super().__init__(cfg, precision=precision, device=device)
        self.fft_len = _next_pow2(int(self.lengths[0]))

    def batch(self, x: torch.Tensor, output: str = "magnitude"):
        _check_freq_pad(x.shape[-1], self.fft_len, self.cfg.pad_mode)
        return super().batch(x, output)


class Cqt2010(Cqt2010v2):
    """transforms.py:326-337 -- the octave recursion with each octave's conv
    through the frequency domain; computed by its time-domain equivalent (see
    Cqt1992), with the frequency route's per-octave fft_len // 2 pad checked."""

    def __init__(self, cfg: CqtConfig, device="cuda"):
        super().__init__(cfg, device=device)
        self.fft_len = _cqt2010_fft_len(cfg, self.early_stages, self.first_bin)

    def batch(self, x: torch.Tensor, output: str = "magnitude"):
        _check_cqt2010_freq_pad(x.shape[-1], self.cfg.pad_mode, self.early_stages, self.n_octaves, self.fft_len)
        return super().batch(x, output)


def _cqt2010_fft_len(cfg: CqtConfig, early_stages: int, first_bin: int) -> int:
    """fft_len of the top-octave bank (kernels.py:383): next power of two >= its longest kernel."""
    n0 = math.ceil(banks.cqt_q(cfg.bins_per_octave) * (cfg.sr / 2 ** early_stages)
                   / (cfg.fmin * 2.0 ** (first_bin / cfg.bins_per_octave)))
    return _next_pow2(int(n0))


def _check_cqt2010_freq_pad(length: int, pad_mode: str, early_stages: int, n_octaves: int, fft_len: int) -> None:
    n = length
    for _ in range(early_stages):
        n = (n + 1) // 2
    for a in range(n_octaves):
        if a > 0:
            n = (n + 1) // 2
        _check_freq_pad(n, fft_len, pad_mode)


def _check_freq_pad(length: int, fft_len: int, pad_mode: str) -> None:
    """signal.py:147-150 for the frequency route's fft_len // 2 centre pad."""
    if pad_mode == "reflect" and fft_len // 2 >= length:
        raise ValueError(f"reflect padding of {fft_len // 2} needs a signal longer than the pad (got {length})")


def stft(x: Signal, params: StftParams | None = None) -> Spectrogram:
    """transforms.py:340-342."""
    return Stft(params or StftParams(), x.sample_rate)(x)


def mel_spectrogram(x: Signal, params: MelParams | None = None) -> Spectrogram:
    """transforms.py:345-347."""
    return MelSpec(params or MelParams(), x.sample_rate)(x)


def cqt1992v2(x: Signal, cfg: CqtConfig, output: str = "magnitude") -> Spectrogram:
    """transforms.py:355-357."""
    return Cqt1992v2(cfg)(x, output)


def cqt2010v2(x: Signal, cfg: CqtConfig, output: str = "magnitude") -> Spectrogram:
    """transforms.py:365-367."""
    return Cqt2010v2(cfg)(x, output)


def cqt1992(x: Signal, cfg: CqtConfig, output: str = "magnitude") -> Spectrogram:
    return Cqt1992(cfg)(x, output)


def cqt2010(x: Signal, cfg: CqtConfig, output: str = "magnitude") -> Spectrogram:
    return Cqt2010(cfg)(x, output)


def batch_transform(signals, transform, threads: int | None = None) -> list:
    """transforms.py:370-388 -- ordered map over clips sharing one sample rate.

    Device transforms run every equal-length group as ONE batched launch;
    `threads` is accepted for signature compatibility (the GPU is the pool).
    Other callables fall back to the plain ordered map."""
    signals = list(signals)
    if not signals:
        return []
    rates = {s.sample_rate for s in signals}
    if len(rates) > 1:
        raise ValueError(f"signals must share one sample rate, got {sorted(rates)}")
    if not isinstance(transform, _Batched):
        return [transform(s) for s in signals]
    for s in signals:
        transform._check_signal(s)
    out = [None] * len(signals)
    groups: dict[int, list[int]] = {}
    for i, s in enumerate(signals):
        groups.setdefault(len(s), []).append(i)
    for idx in groups.values():
        data, meta = transform.batch(torch.stack([signals[i].samples for i in idx]))
        for j, i in enumerate(idx):
            out[i] = Spectrogram(data=data[j], **meta)
    return out


# ---------------------------------------------------------------------------
# trainable layers (gradients.py:28-149)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class DftKernelBank:
    """kernels.py:108-146 -- paired cos/sin rows (n_bins, n_fft)."""

    h_re: np.ndarray
    h_im: np.ndarray


@dataclass(frozen=True)
class MelFilterBank:
    """kernels.py:186-211 -- triangular weights (n_mels, n_fft//2 + 1)."""

    weights: np.ndarray


@dataclass(frozen=True)
class CqtKernelBank:
    """kernels.py:324-358 -- complex time-domain rows (n_bins, width)."""

    time_kernels: np.ndarray


@dataclass
class TrainableLayer:
    """gradients.py:28-100 -- a spectrogram layer with writable kernels.

    Parameters live on the device (`params()` returns the CUDA tensors); the
    forward/backward run batched on the sm_100a kernels (autograd.DftLayerOp).
    """

    kernels: object
    hop: int
    trainable: bool = True
    eps_mag: float = 1e-12
    center: bool = True
    pad_mode: str = "reflect"
    stft_bank: DftKernelBank | None = None
    precision: str = "fp32"
    device: str = "cuda"
    _params: dict = field(init=False, repr=False)

    def __post_init__(self):
        from .autograd import DftLayerOp
        dev = _require_cuda(self.device)
        bank = self.kernels
        if isinstance(bank, DftKernelBank):
            re, im = bank.h_re, bank.h_im
            self._params = {"h_re": torch.tensor(re, dtype=torch.float32, device=dev),
                            "h_im": torch.tensor(im, dtype=torch.float32, device=dev)}
        elif isinstance(bank, CqtKernelBank):
            re, im = bank.time_kernels.real, bank.time_kernels.imag
            self._params = {"h_re": torch.tensor(re, dtype=torch.float32, device=dev),
                            "h_im": torch.tensor(im, dtype=torch.float32, device=dev)}
        elif isinstance(bank, MelFilterBank):
            if self.stft_bank is None:
                raise ValueError("a Mel layer needs the fixed stft_bank it is applied to")
            re, im = self.stft_bank.h_re, self.stft_bank.h_im
            self._params = {"weights": torch.tensor(bank.weights, dtype=torch.float32, device=dev)}
        else:
            raise TypeError(f"unsupported kernel bank type {type(bank).__name__}")
        self._op = DftLayerOp(re, im, self.hop, self.center, self.pad_mode, self.eps_mag, self.precision, dev)
        self._fixed = (torch.tensor(re, dtype=torch.float32, device=dev),
                       torch.tensor(im, dtype=torch.float32, device=dev))

    def params(self) -> dict:
        return self._params

    @property
    def is_mel(self) -> bool:
        return isinstance(self.kernels, MelFilterBank)

    def _bank(self):
        if self.is_mel:
            return self._fixed
        return self._params["h_re"], self._params["h_im"]

    def _run(self, x: torch.Tensor, for_vjp: bool = False):
        h_re, h_im = self._bank()
        self._op.set_bank(h_re, h_im)
        # a convolution layer's VJP weighs every frame by the phasor re/S, im/S: its
        # forward runs split-precision (autograd.DftLayerOp, phasor="split")
        return self._op.forward(x, self._params["weights"] if self.is_mel else None,
                                phasor_grads=for_vjp and not self.is_mel)

    def spectrogram_batch(self, x: torch.Tensor) -> torch.Tensor:
        """(B, L) -> (B, bins, frames) smoothed magnitude (or W @ it)."""
        return self._run(x)[0]

    def spectrogram(self, x: Signal) -> torch.Tensor:
        return self.spectrogram_batch(x.samples[None])[0]


def spectrogram_vjp(x, layer: TrainableLayer, upstream_grad, with_input_grad: bool = False):
    """gradients.py:103-149 -- pull a loss gradient back onto the kernels.

    `x` is a Signal (one clip, as the reference) or a (B, L) tensor (batch:
    the kernel gradients are summed over the clips).  Returns a dict keyed
    like layer.params(); with_input_grad adds dL/dx (conv layers only)."""
    xs = x.samples[None] if isinstance(x, Signal) else _batch(x)
    g = torch.as_tensor(np.asarray(upstream_grad) if not torch.is_tensor(upstream_grad) else upstream_grad)
    g = g.to(layer._op.device, torch.float32)
    out, saved = layer._run(xs, for_vjp=True)
    if g.dim() == 2:
        g = g[None]
    if tuple(g.shape) != tuple(out.shape):
        raise ValueError(f"upstream_grad shape {tuple(g.shape)} != spectrogram shape {tuple(out.shape)}")
    if layer.is_mel:
        if with_input_grad:
            raise NotImplementedError("input gradients are only provided for convolution layers")
        gr = layer._op.backward(saved, g, mel_w=layer._params["weights"], need_bank=False, need_mel=True)
        return {"weights": gr["weights"]}
    h_re, h_im = layer._bank()
    gr = layer._op.backward(saved, g, h_re, h_im, need_bank=True, need_x=with_input_grad)
    grads = {"h_re": gr["h_re"], "h_im": gr["h_im"]}
    if not with_input_grad:
        return grads
    gx = gr["x"]
    return grads, (gx[0] if isinstance(x, Signal) else gx)


def _batch(x):
    x = x if torch.is_tensor(x) else torch.as_tensor(np.asarray(x, dtype=np.float32))
    return x[None] if x.dim() == 1 else x
