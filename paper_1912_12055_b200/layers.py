"""nnAudio-style nn.Modules on the sm_100a kernels.

    STFT(n_fft=2048, freq_bins=None, hop_length=512, window='hann', freq_scale='no', center=True,
         pad_mode='reflect', fmin=50, fmax=6000, sr=22050, trainable=False, output_format='Magnitude')
    MelSpectrogram(sr=22050, n_fft=2048, n_mels=128, hop_length=512, window='hann', center=True,
         pad_mode='reflect', htk=False, fmin=0.0, fmax=None, norm=None, power=1.0,
         trainable_mel=False, trainable_STFT=False)
    CQT1992v2(sr=22050, hop_length=512, fmin=32.70, fmax=None, n_bins=84, bins_per_octave=12, norm=1,
         window='hann', center=True, pad_mode='reflect', trainable=False, output_format='Magnitude')
    CQT2010v2(sr=22050, hop_length=512, fmin=32.70, fmax=None, n_bins=84, bins_per_octave=12, norm=True,
         basis_norm=1, window='hann', pad_mode='reflect', earlydownsample=True)
    CQT1992, CQT2010: the frequency-domain variants (same arguments as the v2 modules),
         computed by their time-domain equivalents (spectro.Cqt1992 / Cqt2010)

Input (batch, samples) or (samples,) float32 CUDA tensor; output (batch, freq, time).
precision: "tf32" (default) / "f16" (FP16 operands under exact power-of-two scales,
the same <= 1e-3 accuracy at twice the tensor rate; STFT / Mel inference) / "fp32"
(<= 1e-5).  grad_phasor (trainable STFT / Mel): "split" (default) computes the
forward that saves the phasor re/S, im/S split-precision so TF32 kernel / input
gradients meet 2e-3; "tf32" keeps the one-pass forward (faster, gradient tail
up to ~1e-1 where |X| is near zero).
Numerics follow the `spectro` reference this repo is parity-checked against:
Mel `norm=None` is its peak normalisation (spectro MelParams norm="none"); nnAudio's
`norm=1` selects the area ("slaney") normalisation.  Trainable layers return the
smoothed magnitude sqrt(re^2 + im^2 + 1e-12) of gradients.py:61-67 and back-propagate
through tcgen05 GEMMs (autograd.py).  Inference layers never touch the CPU.
"""

from __future__ import annotations

import torch
from torch import nn

from . import banks
from .autograd import DftLayerFunction, DftLayerOp
from .engine import CqtLongEngine, Cqt2010Engine, DftEngine, _require_cuda
from .spectro import CqtConfig, cqt2010_plan

_FORMATS = {"magnitude": "magnitude", "complex": "complex", "power": "power"}


def _fmt(output_format: str) -> str:
    k = output_format.lower()
    if k not in _FORMATS:
        raise ValueError(f"output_format must be one of Magnitude/Complex/Power, got {output_format!r}")
    return _FORMATS[k]


def _train_prec(precision: str) -> str:
    """The autograd path's GEMMs take TF32 operands: FP16 inference modes train in
    the TF32 mode of the same accuracy."""
    return {"f16": "tf32", "3xf16": "fp32"}.get(precision, precision)


def _bank_key(*ps):
    return tuple((p.data_ptr(), p._version) for p in ps)


def _as_batch(x: torch.Tensor) -> torch.Tensor:
    if x.dim() == 1:
        return x[None]
    if x.dim() == 3 and x.shape[1] == 1:  # (batch, 1, len), nnAudio accepts it
        return x[:, 0]
    if x.dim() != 2:
        raise ValueError(f"expected (batch, len) audio, got {tuple(x.shape)}")
    return x


class STFT(nn.Module):
    def __init__(self, n_fft=2048, freq_bins=None, hop_length=512, window="hann", freq_scale="no", center=True,
                 pad_mode="reflect", fmin=50, fmax=6000, sr=22050, trainable=False, output_format="Magnitude",
                 precision="tf32", device="cuda", log_eps=None, grad_phasor="split"):
        super().__init__()
        self.device = _require_cuda(device)
        self.output_format = _fmt(output_format)
        # log_eps: log(|X| + log_eps) (or of the power) fused into the epilogue (extension,
        # north_star item 3); the trainable path composes torch.log on the kernel output
        self.log_eps = log_eps
        self.trainable = bool(trainable)
        nf, self.bin_freqs_hz = banks.frequency_scale(freq_scale, n_fft, sr, fmin, fmax, freq_bins)
        h_re, h_im = banks.dft_kernels(nf, banks.make_window(window, n_fft, True))
        self.h_re = nn.Parameter(torch.tensor(h_re, dtype=torch.float32, device=self.device), requires_grad=trainable)
        self.h_im = nn.Parameter(torch.tensor(h_im, dtype=torch.float32, device=self.device), requires_grad=trainable)
        self._infer = DftEngine(h_re, h_im, hop_length, center, pad_mode, precision=precision, device=self.device)
        self._op = DftLayerOp(h_re, h_im, hop_length, center, pad_mode, precision=_train_prec(precision),
                              device=self.device, phasor=grad_phasor)
        self._op._bank_version = None
        self._infer_key = _bank_key(self.h_re, self.h_im)

    def forward(self, x: torch.Tensor, output_format: str | None = None) -> torch.Tensor:
        x = _as_batch(x)
        fmt = _fmt(output_format or self.output_format)
        if self.trainable or x.requires_grad:
            # autograd path: the smoothed magnitude S = sqrt(|X|^2 + 1e-12) of gradients.py:61-67;
            # power is S^2 through autograd, complex output has no reference VJP
            if fmt == "complex":
                raise NotImplementedError("trainable / input-gradient STFT supports Magnitude and Power outputs "
                                          "(the reference VJP is for the smoothed magnitude, gradients.py:103-149)")
            y = DftLayerFunction.apply(x, self.h_re, self.h_im, None, self._op, _bank_key(self.h_re, self.h_im))
            if fmt == "power":
                y = y * y
            return y if self.log_eps is None else torch.log(y + self.log_eps)
        key = _bank_key(self.h_re, self.h_im)
        if key != self._infer_key:  # parameters replaced / edited in place (load_state_dict, optimiser step)
            self._infer.set_bank(self.h_re.detach(), self.h_im.detach())
            self._infer_key = key
        if self.log_eps is not None and fmt != "complex":
            return self._infer.forward(x, fmt, log_eps=self.log_eps)
        return self._infer.forward(x, fmt)


class MelSpectrogram(nn.Module):
    def __init__(self, sr=22050, n_fft=2048, n_mels=128, hop_length=512, window="hann", center=True,
                 pad_mode="reflect", htk=False, fmin=0.0, fmax=None, norm=None, power=1.0, trainable_mel=False,
                 trainable_STFT=False, precision="tf32", device="cuda", log_eps=None, grad_phasor="split"):
        super().__init__()
        self.device = _require_cuda(device)
        self.log_eps = log_eps  # log(mel + log_eps) fused into the epilogue (extension, north_star item 3)
        nf, _ = banks.frequency_scale("no", n_fft, sr, 50.0, 6000.0, None)
        h_re, h_im = banks.dft_kernels(nf, banks.make_window(window, n_fft, True))
        mel_norm = {None: "none", "none": "none", 1: "area", "slaney": "area", "area": "area"}[norm]
        w, self.mel_center_freqs_hz = banks.mel_filter_bank(sr, n_fft, n_mels, fmin=fmin, fmax=fmax,
                                                            formula="htk" if htk else "slaney", norm=mel_norm)
        self.power = float(power)
        self.trainable_mel, self.trainable_STFT = bool(trainable_mel), bool(trainable_STFT)
        self.mel_basis = nn.Parameter(torch.tensor(w, dtype=torch.float32, device=self.device),
                                      requires_grad=trainable_mel)
        self.h_re = nn.Parameter(torch.tensor(h_re, dtype=torch.float32, device=self.device),
                                 requires_grad=trainable_STFT)
        self.h_im = nn.Parameter(torch.tensor(h_im, dtype=torch.float32, device=self.device),
                                 requires_grad=trainable_STFT)
        self._infer = DftEngine(h_re, h_im, hop_length, center, pad_mode, precision=precision, device=self.device)
        self._infer.set_mel(w, power=self.power)
        self._op = DftLayerOp(h_re, h_im, hop_length, center, pad_mode, precision=_train_prec(precision),
                              device=self.device, phasor=grad_phasor)
        self._op._bank_version = None
        self._infer_key = _bank_key(self.h_re, self.h_im, self.mel_basis)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        x = _as_batch(x)
        if self.trainable_mel or self.trainable_STFT or x.requires_grad:
            if self.power != 1.0:
                raise NotImplementedError("trainable Mel layers use power=1 (gradients.py:69-80)")
            y = DftLayerFunction.apply(x, self.h_re, self.h_im, self.mel_basis, self._op,
                                       _bank_key(self.h_re, self.h_im))
            return y if self.log_eps is None else torch.log(y + self.log_eps)
        key = _bank_key(self.h_re, self.h_im, self.mel_basis)
        if key != self._infer_key:  # parameters edited in place since construction
            self._infer.set_bank(self.h_re.detach(), self.h_im.detach())
            self._infer.set_mel(self.mel_basis.detach(), power=self.power)
            self._infer_key = key
        return self._infer.forward(x, "mel", log_eps=self.log_eps)


class CQT1992v2(nn.Module):
    def __init__(self, sr=22050, hop_length=512, fmin=32.70, fmax=None, n_bins=84, bins_per_octave=12, norm=1,
                 window="hann", center=True, pad_mode="reflect", trainable=False, output_format="Magnitude",
                 precision="tf32", device="cuda"):
        super().__init__()
        if not center:
            raise NotImplementedError("CQT1992v2 frames are centred (transforms.py:175-186)")
        self.device = _require_cuda(device)
        self.cfg = CqtConfig(sr=sr, fmin=fmin, n_bins=n_bins, bins_per_octave=bins_per_octave,
                             hop_length=hop_length, window_kind=window, norm=norm, fmax=fmax, pad_mode=pad_mode)
        k, self.lengths = banks.cqt_time_kernels(sr, self.cfg.bin_freqs_hz, bins_per_octave, window, norm)
        self.output_format = _fmt(output_format)
        self.trainable = bool(trainable)
        self.k_re = nn.Parameter(torch.tensor(k.real, dtype=torch.float32, device=self.device),
                                 requires_grad=trainable)
        self.k_im = nn.Parameter(torch.tensor(k.imag, dtype=torch.float32, device=self.device),
                                 requires_grad=trainable)
        self._infer = CqtLongEngine(k, hop_length, pad_mode, precision=precision, device=self.device)
        self._op = None
        self._precision = precision
        self._infer_key = _bank_key(self.k_re, self.k_im)

    def forward(self, x: torch.Tensor, output_format: str | None = None) -> torch.Tensor:
        x = _as_batch(x)
        if self.trainable or x.requires_grad:
            if self._op is None:  # dense DFT-layout op over the CQT rows (trainable rows lose their support)
                self._op = DftLayerOp(self.k_re.detach(), self.k_im.detach(), self.cfg.hop_length, True,
                                      self.cfg.pad_mode, precision=_train_prec(self._precision), device=self.device)
                self._op._bank_version = None
            if _fmt(output_format or self.output_format) != "magnitude":
                raise NotImplementedError("trainable CQT1992v2 returns the smoothed magnitude (gradients.py:61-67)")
            return DftLayerFunction.apply(x, self.k_re, self.k_im, None, self._op, _bank_key(self.k_re, self.k_im))
        key = _bank_key(self.k_re, self.k_im)
        if key != self._infer_key:  # parameters replaced / edited in place: repack bank + schedule
            self._infer.set_bank(self.k_re.detach().cpu().numpy(), self.k_im.detach().cpu().numpy())
            self._infer_key = key
        return self._infer.forward(x, _fmt(output_format or self.output_format))


class CQT2010v2(nn.Module):
    def __init__(self, sr=22050, hop_length=512, fmin=32.70, fmax=None, n_bins=84, bins_per_octave=12, norm=True,
                 basis_norm=1, window="hann", pad_mode="reflect", earlydownsample=True, output_format="Magnitude",
                 device="cuda"):
        super().__init__()
        if norm is not True and norm != 1:
            # the reference's Cqt2010v2 output has one scaling (transforms.py:290-313): L1-normalised
            # kernels via basis_norm, no further output normalisation to switch off
            raise NotImplementedError("CQT2010v2 supports norm=True only (the reference's output scaling)")
        self.device = _require_cuda(device)
        self.cfg = CqtConfig(sr=sr, fmin=fmin, n_bins=n_bins, bins_per_octave=bins_per_octave,
                             hop_length=hop_length, window_kind=window, norm=basis_norm, fmax=fmax,
                             pad_mode=pad_mode, early_downsample=earlydownsample)
        p = cqt2010_plan(self.cfg)
        self.output_format = _fmt(output_format)
        self._eng = Cqt2010Engine(p["taps"], p["top_kernels"], p["early_stages"], p["n_octaves"], p["kernel_hop"],
                                  p["first_bin"], bins_per_octave, self.cfg.n_bins, pad_mode, device=self.device)

    def forward(self, x: torch.Tensor, output_format: str | None = None) -> torch.Tensor:
        return self._eng.forward(_as_batch(x), _fmt(output_format or self.output_format))


class CQT1992(CQT1992v2):
    """The frequency-domain CQT (transforms.py:211-238): equal to CQT1992v2 by the
    power theorem; the frequency route's own fft_len // 2 reflect-pad constraint
    is checked (spectro.Cqt1992)."""

    def forward(self, x: torch.Tensor, output_format: str | None = None) -> torch.Tensor:
        from .spectro import _check_freq_pad, _next_pow2
        x = _as_batch(x)
        _check_freq_pad(x.shape[-1], _next_pow2(int(self.lengths[0])), self.cfg.pad_mode)
        return super().forward(x, output_format)


class CQT2010(CQT2010v2):
    """The frequency-domain octave recursion (transforms.py:326-337), computed by
    CQT2010v2's chain; the per-octave fft_len // 2 pad constraint is checked
    (spectro.Cqt2010)."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        from .spectro import _cqt2010_fft_len
        p = cqt2010_plan(self.cfg)
        self._plan = (p["early_stages"], p["n_octaves"], _cqt2010_fft_len(self.cfg, p["early_stages"], p["first_bin"]))

    def forward(self, x: torch.Tensor, output_format: str | None = None) -> torch.Tensor:
        from .spectro import _check_cqt2010_freq_pad
        x = _as_batch(x)
        _check_cqt2010_freq_pad(x.shape[-1], self.cfg.pad_mode, *self._plan)
        return super().forward(x, output_format)
