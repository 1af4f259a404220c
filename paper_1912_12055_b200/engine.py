"""Device-side engines: own the packed kernel banks on the GPU and run the
sm_100a kernels through the C ABI.  Everything above this module (the
`spectro`-compatible transforms and the nnAudio-style nn.Modules) funnels
through here, mirroring how every reference transform funnels through
`conv1d_strided` (signal.py:159-183)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L


def _require_cuda(device) -> torch.device:
    device = torch.device(device)
    if device.type != "cuda":
        raise L.NnabError("paper_1912_12055_b200 runs only on CUDA (sm_100a); got device " + str(device))
    if not torch.cuda.is_available():
        raise L.NnabError("no CUDA device: the sm_100a kernels have no CPU fallback")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    major, _ = torch.cuda.get_device_capability(device)
    if major != 10:
        raise L.NnabError(f"sm_100 (B200) required, found compute capability {major}.x")
    return device


def frames_struct(B: int, length: int, width: int, hop: int, pad: int, pad_mode: str) -> L.nnab_frames:
    if pad_mode not in L.PAD_MODES:
        raise ValueError(f"unknown pad mode {pad_mode!r}")
    return L.nnab_frames(int(B), int(length), int(width), int(hop), int(pad), L.PAD_MODES[pad_mode])


def geometry(length: int, width: int, hop: int, pad: int, pad_mode: str):
    """(n_frames, row_len, rows_per_clip) with the reference's ValueErrors."""
    if hop < 1:
        raise ValueError(f"stride must be >= 1, got {hop}")
    if pad_mode == "reflect" and pad > 0 and pad >= length:
        raise ValueError(f"reflect padding ({pad}, {pad}) must be shorter than the signal (len {length})")
    if width > length + 2 * pad:
        raise ValueError(f"kernel length {width} exceeds signal length {length + 2 * pad}; pad the signal first")
    f = frames_struct(1, length, width, hop, pad, pad_mode)
    t, rl, r = C.c_int32(), C.c_int32(), C.c_int32()
    L.check(L.load().nnab_frames_geometry(C.byref(f), C.byref(t), C.byref(rl), C.byref(r)), "frames_geometry")
    return t.value, rl.value, r.value


class _Workspace:
    """Grow-only device scratch, one per engine and device."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        return self.buf


class DftEngine:
    """A DFT-type bank (h_re, h_im rows of width n_fft) applied at a hop,
    optionally followed by a fused Mel projection.

    fold_nyquist packs the default integer-bin bank into whole 256-row tiles
    (its bin-0 and Nyquist sine rows are zero); trainable banks never fold
    because their sine rows may become non-zero.
    """

    # "fp32" on this engine: the FP16 hi/lo split (same <= 1e-5 accuracy as 3xTF32, 2x the MMA rate)
    FP32_MODE = L.PREC_3XF16

    def __init__(self, h_re, h_im, hop: int, center: bool = True, pad_mode: str = "reflect",
                 precision: str = "tf32", device="cuda", allow_fold: bool = True, f16_ok: bool = True):
        self.device = _require_cuda(device)
        if precision not in L.PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(L.PRECISIONS)}")
        self.precision = L.PRECISIONS[precision]
        if precision == "fp32" and f16_ok:
            self.precision = self.FP32_MODE
        if not f16_ok and self.precision in (L.PREC_F16, L.PREC_3XF16):
            raise ValueError("this layer supports precision 'tf32' or 'fp32' (3xTF32)")
        h_re = torch.as_tensor(h_re)
        h_im = torch.as_tensor(h_im)
        if h_re.shape != h_im.shape or h_re.dim() != 2:
            raise ValueError("h_re and h_im must be equal-shape 2-D banks")
        self.n_bins, self.n_fft = int(h_re.shape[0]), int(h_re.shape[1])
        self.hop, self.center, self.pad_mode = int(hop), bool(center), pad_mode
        if self.hop < 1:
            raise ValueError(f"stride must be >= 1, got {hop}")
        self.fold = 0
        # allow_fold="exact" (trainable banks): fold only while the bin-0 and Nyquist sine rows are
        # zero to 1e-9 of the bank's peak (sin(pi k) rounding), re-checked at every set_bank; their
        # gradients are as small (im ~ 0 makes coef_im ~ 0, gradients.py:127-129), so training
        # keeps them there
        self._fold_exact = allow_fold == "exact"
        if allow_fold and not self._fold_exact and self.n_bins >= 2:
            scale = float(h_re.abs().max()) or 1.0
            z0 = float(h_im[0].abs().max()) <= 1e-9 * scale
            zn = float(h_im[-1].abs().max()) <= 1e-9 * scale
            self.fold = int(z0 and zn and (self.n_bins - 1) % 128 == 0)
        self._ws = _Workspace()
        self.mel_w = None
        self.mel_wide = False
        self.set_bank(h_re, h_im)

    # ------------------------------------------------------------ banks
    def set_bank(self, h_re, h_im) -> None:
        """(Re)pack the bank on the device (used every step by trainable layers)."""
        lib = L.load()
        h_re = torch.as_tensor(h_re).to(self.device, torch.float32).contiguous()
        h_im = torch.as_tensor(h_im).to(self.device, torch.float32).contiguous()
        self._bank = (h_re, h_im)
        if self._fold_exact:  # one read back per repack
            self.fold = int(self.n_bins >= 2 and (self.n_bins - 1) % 128 == 0 and
                            bool(h_im[[0, -1]].abs().amax() <= 1e-9 * h_re.abs().amax()))
        nbytes = lib.nnab_dft_bank_bytes_prec(self.n_bins, self.n_fft, self.fold, self.precision)
        n = nbytes // 4
        if getattr(self, "packed_hi", None) is None or self.packed_hi.numel() != n:
            self.packed_hi = torch.empty(n, dtype=torch.float32, device=self.device)
            self.packed_lo = (torch.empty(n, dtype=torch.float32, device=self.device)
                              if self.precision in (L.PREC_3XTF32, L.PREC_3XF16) else None)
        L.check(lib.nnab_pack_dft_bank(h_re.data_ptr(), h_im.data_ptr(), self.n_bins, self.n_fft, self.fold,
                                       self.precision, self.packed_hi.data_ptr(), L.ptr(self.packed_lo),
                                       L.stream_handle(self.device)), "pack_dft_bank")
        self.n_tiles = lib.nnab_dft_bank_tiles(self.n_bins, self.fold)

    def set_mel(self, weights, power: float = 1.0, banded: bool = True) -> None:
        """Mel weights (n_mels, n_bins) for the fused epilogue; rows padded to
        a multiple of 4 floats so the epilogue reads them with 16-byte loads.
        More than 128 mel rows (the epilogue's shared-memory accumulator) run
        as the STFT GEMM saving |X| per frame slot, then a tcgen05 W @ |X| GEMM
        (power 1, no fused log)."""
        w = torch.as_tensor(weights)
        if w.dim() != 2 or w.shape[1] != self.n_bins:
            raise ValueError(f"mel weights must be (n_mels, {self.n_bins})")
        self.n_mels = int(w.shape[0])
        self.power = float(power)
        self.mel_wide = self.n_mels > 128
        if self.mel_wide:
            if self.precision in (L.PREC_F16, L.PREC_3XF16):  # the slot GEMMs take TF32 operands
                self.precision = L.PREC_TF32 if self.precision == L.PREC_F16 else L.PREC_3XTF32
                self.set_bank(*self._bank)
            kp = (self.n_bins + 31) // 32 * 32
            wp = torch.zeros(self.n_mels, kp, dtype=torch.float32, device=self.device)
            wp[:, : self.n_bins] = w.to(self.device, torch.float32)
            self.mel_w = wp
            self.mel_ld, self.mel_band = kp, None
            return
        self.mel_ld = ((max(self.n_tiles * 128, self.n_bins) + 3) // 4) * 4 + 32
        wp = torch.zeros(self.n_mels, self.mel_ld, dtype=torch.float32, device=w.device)
        wp[:, : self.n_bins] = w.to(torch.float32)
        self.mel_w = wp.to(self.device)
        n_chunks = self.mel_ld // 32 + 1
        if banded:
            from .banks import mel_bands
            band = mel_bands(wp.cpu().numpy(), n_chunks)
            self.mel_band = torch.from_numpy(band.reshape(-1)).to(self.device)
        else:
            self.mel_band = None

    def _split(self, t: torch.Tensor):
        """TF32-round t (hi), plus the residual (lo) in 3xTF32 mode."""
        lib = L.load()
        hi = torch.empty_like(t)
        lo = torch.empty_like(t) if self.precision == L.PREC_3XTF32 else None
        L.check(lib.nnab_tf32_split(t.data_ptr(), t.numel(), self.precision, hi.data_ptr(), L.ptr(lo),
                                    L.stream_handle(self.device)), "tf32_split")
        return hi, lo

    def _mel_wide(self, B: int, length: int, out: torch.Tensor, log_flag: int) -> torch.Tensor:
        """n_mels > 128: |X| per (bin, frame slot) from the STFT GEMM, then W @ |X|."""
        if self.power != 1.0 or log_flag:
            raise NotImplementedError("more than 128 mel rows support power=1 without fused log compression")
        lib = L.load()
        f = self.frames(B, length)
        ws, stream, dev = self._ws.buf, L.stream_handle(self.device), self.device
        split = self.precision == L.PREC_3XTF32
        ld = lib.nnab_slots_ld(C.byref(f))
        F = self.n_bins
        pad = self.n_fft // 2 if self.center else 0
        T, _, R = geometry(length, self.n_fft, self.hop, pad, self.pad_mode)
        re = torch.empty(F, ld, device=dev)
        im = torch.empty(F, ld, device=dev) if split else None
        mag = torch.empty(F, ld, device=dev)
        L.check(lib.nnab_stft_forward_train_staged(
            C.byref(f), self.packed_hi.data_ptr(), L.ptr(self.packed_lo), F, self.fold, self.precision,
            L.OUT_SMOOTH_MAG, 1.0, 0.0, None, 0, 0, None, None, re.data_ptr(), L.ptr(im), mag.data_ptr(), ld,
            ws.data_ptr(), ws.numel(), stream), "stft_forward_train_staged")
        del re, im
        kp = self.mel_ld
        w_hi, w_lo = self._split(self.mel_w)
        m_hi, m_lo = self._split(mag) if split else (mag, None)
        rc = lib.nnab_mel_forward_slots(self.n_mels, ld, kp, w_hi.data_ptr(), L.ptr(w_lo), m_hi.data_ptr(),
                                        L.ptr(m_lo), F, B, R, T, self.precision, out.data_ptr(), stream)
        if rc == L.ENOTSUP or (rc == L.EINVAL and R % 4):  # slot-major W @ |X|, then the (B, n_mels, T) layout
            mel_s = torch.empty(self.n_mels, ld, device=dev)
            part = torch.empty(max(lib.nnab_rgemm_partial_bytes(self.n_mels, ld, kp, 1) // 4, 1), device=dev)
            L.check(lib.nnab_rgemm(self.n_mels, ld, kp, w_hi.data_ptr(), L.ptr(w_lo), kp, m_hi.data_ptr(),
                                   L.ptr(m_lo), ld, 1, ld, F, mel_s.data_ptr(), ld, 1, part.data_ptr(),
                                   self.precision, stream), "rgemm")
            L.check(lib.nnab_from_slots(mel_s.data_ptr(), B, self.n_mels, T, R, ld, out.data_ptr(), stream),
                    "from_slots")
        else:
            L.check(rc, "mel_forward_slots")
        return out

    # ------------------------------------------------------------ forward
    def frames(self, B: int, length: int) -> L.nnab_frames:
        pad = self.n_fft // 2 if self.center else 0
        return frames_struct(B, length, self.n_fft, self.hop, pad, self.pad_mode)

    def n_frames(self, length: int) -> int:
        pad = self.n_fft // 2 if self.center else 0
        return geometry(length, self.n_fft, self.hop, pad, self.pad_mode)[0]

    def forward(self, x: torch.Tensor, kind: str = "magnitude", eps: float | None = None,
                out: torch.Tensor | None = None, log_eps: float | None = None) -> torch.Tensor:
        """x (B, L) float32 on the engine's device -> (B, F, T) [complex64 for 'complex',
        (B, n_mels, T) for 'mel'].  eps only enters 'smooth' (sqrt(|X|^2 + eps),
        default 1e-12, gradients.py:61-67) and 'mel' (default 0: MelSpec is
        W @ |X|**power with the plain magnitude, transforms.py:164-172).  log_eps
        (magnitude / power / mel): the epilogue writes log(value + log_eps)."""
        B, length = self.stage(x)
        return self.run_staged(B, length, kind, eps, out, log_eps)

    _KINDS = {"magnitude": L.OUT_MAGNITUDE, "power": L.OUT_POWER, "complex": L.OUT_COMPLEX,
              "mel": L.OUT_MEL, "smooth": L.OUT_SMOOTH_MAG}

    def stage(self, x: torch.Tensor):
        """Pad + lay out x as hop rows in the engine workspace (nnab_stage_frames).
        Returns (B, L); the staged frames stay valid until the next stage()."""
        lib = L.load()
        if x.dim() == 1:
            x = x[None]
        if x.device != self.device:
            raise ValueError(f"input on {x.device}, engine on {self.device}")
        x = x.to(torch.float32).contiguous()
        B, length = int(x.shape[0]), int(x.shape[1])
        if length < 1:
            raise ValueError("signal must be non-empty")
        self.n_frames(length)  # reference ValueErrors before any launch
        if B == 0:
            return B, length
        f = self.frames(B, length)
        ws = self._ws.get(lib.nnab_stft_workspace_bytes(C.byref(f), self.precision), self.device)
        L.check(lib.nnab_stage_frames(C.byref(f), x.data_ptr(), self.precision, ws.data_ptr(), ws.numel(),
                                      L.stream_handle(self.device)), "stage_frames")
        return B, length

    def run_staged(self, B: int, length: int, kind: str = "magnitude", eps: float | None = None,
                   out: torch.Tensor | None = None, log_eps: float | None = None) -> torch.Tensor:
        """The tcgen05 GEMM + fused epilogue on the frames staged by stage()."""
        lib = L.load()
        if eps is None:
            eps = 1e-12 if kind == "smooth" else 0.0
        log_flag = 0
        if log_eps is not None:
            if kind not in ("magnitude", "power", "mel"):
                raise ValueError("log compression applies to magnitude, power and mel outputs")
            if not log_eps >= 0.0:
                raise ValueError(f"log_eps must be >= 0, got {log_eps}")
            log_flag, eps = L.OUT_LOG, float(log_eps)
        T = self.n_frames(length)
        if kind not in self._KINDS:
            raise ValueError(f"output must be one of {sorted(self._KINDS)}, got {kind!r}")
        k = self._KINDS[kind]
        if k == L.OUT_MEL and self.mel_w is None:
            raise ValueError("set_mel() first")
        if out is None:
            rows = self.n_mels if k == L.OUT_MEL else self.n_bins
            dt = torch.complex64 if k == L.OUT_COMPLEX else torch.float32
            out = torch.empty(B, rows, T, dtype=dt, device=self.device)
        if B == 0:
            return out
        mel = k == L.OUT_MEL
        if mel and self.mel_wide:
            return self._mel_wide(B, length, out, log_flag)
        f = self.frames(B, length)
        ws = self._ws.buf
        L.check(lib.nnab_stft_forward_staged(
            C.byref(f), self.packed_hi.data_ptr(), L.ptr(self.packed_lo), self.n_bins, self.fold,
            self.precision, k | log_flag, float(getattr(self, "power", 1.0)), float(eps),
            self.mel_w.data_ptr() if mel else None, self.n_mels if mel else 0, self.mel_ld if mel else 0,
            L.ptr(self.mel_band) if mel else None, out.data_ptr(), ws.data_ptr(), ws.numel(),
            L.stream_handle(self.device)), "stft_forward_staged")
        return out

    def forward_host(self, x_host: torch.Tensor, kind: str = "magnitude", chunk_clips: int = 128,
                     out_host: torch.Tensor | None = None, log_eps: float | None = None) -> torch.Tensor:
        """Pinned host (B, L) -> pinned host result, streamed through the GPU
        in chunks with copy/compute overlap (nnab_stft_forward_host)."""
        lib = L.load()
        B, length = int(x_host.shape[0]), int(x_host.shape[1])
        T = self.n_frames(length)
        k = {"magnitude": L.OUT_MAGNITUDE, "power": L.OUT_POWER, "mel": L.OUT_MEL}[kind]
        if k == L.OUT_MEL and self.mel_wide:
            raise NotImplementedError("the host-buffer entry point fuses at most 128 mel rows")
        rows = self.n_mels if k == L.OUT_MEL else self.n_bins
        if out_host is None:
            out_host = torch.empty(B, rows, T, dtype=torch.float32, pin_memory=True)
        f = self.frames(B, length)
        need = lib.nnab_stft_host_scratch_bytes(C.byref(f), self.precision, rows, chunk_clips)
        ws = self._ws.get(need, self.device)
        mel = k == L.OUT_MEL
        L.check(lib.nnab_stft_forward_host(
            C.byref(f), x_host.data_ptr(), self.packed_hi.data_ptr(), L.ptr(self.packed_lo), self.n_bins, self.fold,
            self.precision, k | (L.OUT_LOG if log_eps is not None else 0), float(getattr(self, "power", 1.0)),
            float(log_eps) if log_eps is not None else 0.0,
            self.mel_w.data_ptr() if mel else None, self.n_mels if mel else 0, self.mel_ld if mel else 0,
            L.ptr(self.mel_band) if mel else None, out_host.data_ptr(), int(chunk_clips), ws.data_ptr(),
            ws.numel(), L.stream_handle(self.device)), "stft_forward_host")
        return out_host


def _row_support(k_re: np.ndarray, k_im: np.ndarray) -> np.ndarray:
    """[begin, end) of the non-zero columns of each complex row (int32 pairs)."""
    nz = (k_re != 0) | (k_im != 0)
    sup = np.zeros((k_re.shape[0], 2), dtype=np.int32)
    for r in range(k_re.shape[0]):
        idx = np.flatnonzero(nz[r])
        if idx.size:
            sup[r] = (idx[0], idx[-1] + 1)
    return sup


class CqtLongEngine:
    """CQT1992v2's long complex bank (kernels.py:361-402) on the tcgen05 GEMM.

    method "hybrid" (default; TF32, hop 512): the long low-frequency bins --
    support >= 8 hops -- on the hop-offset E-GEMM (csrc/cqt1992_egemm.cu), the
    rest on the longest-first per-K-block schedule (csrc/cqt1992.cu), from one
    staging of the frames.  "schedule" / "egemm" run one method for every bin;
    3xTF32 always uses the schedule."""

    LONG_HOPS = 3  # hybrid: bins whose support spans >= this many hops go to the E-GEMM (swept: 1.66 ms)

    def __init__(self, kernels, hop: int, pad_mode: str = "reflect", precision: str = "tf32", device="cuda",
                 dense: bool = False, method: str = "hybrid"):
        self.device = _require_cuda(device)
        if precision not in L.PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(L.PRECISIONS)}")
        # "fp32": 3xF16 on the hybrid (E-GEMM + schedule), 3xTF32 for the other methods
        self.precision = L.PRECISIONS[precision]
        if precision == "fp32" and method == "hybrid" and not dense and int(hop) == 512:
            self.precision = L.PREC_3XF16
        if self.precision in (L.PREC_F16, L.PREC_3XF16) and (method != "hybrid" or dense or int(hop) != 512):
            raise ValueError("FP16 operand modes run the hybrid CQT1992v2 (hop 512)")
        k = np.asarray(kernels)
        self.n_bins, self.width = int(k.shape[0]), int(k.shape[1])
        self.hop, self.pad_mode = int(hop), pad_mode
        if method not in ("egemm", "schedule", "hybrid"):
            raise ValueError(f"method must be 'hybrid', 'egemm' or 'schedule', got {method!r}")
        self.method = "schedule" if dense else method
        if self.hop < 1:
            raise ValueError(f"stride must be >= 1, got {hop}")
        self._ws = _Workspace()
        self.set_bank(k.real, k.imag, dense=dense)

    def _schedule(self, sup, dr, di):
        """Per-K-block schedule + packed bank of the rows in dr/di (device) with supports sup."""
        lib = L.load()
        nb = int(sup.shape[0])
        cap = lib.nnab_cqt_bank_tiles(nb) * (((self.width + 63) // 64 * 64) // 16) + 16
        tab = np.zeros(cap, dtype=np.uint32)
        n_ent = C.c_int32()
        L.check(lib.nnab_cqt_schedule(np.ascontiguousarray(sup).ctypes.data, nb, self.width, self.precision,
                                      tab.ctypes.data, C.byref(n_ent)), "cqt_schedule")
        tiles = lib.nnab_cqt_bank_tiles(nb)
        schedule = torch.from_numpy(tab[: tiles * n_ent.value].astype(np.int32)).to(self.device)
        n = lib.nnab_cqt_bank_bytes_prec(nb, self.width, self.precision) // 4
        hi = torch.empty(n, dtype=torch.float32, device=self.device)
        lo = (torch.empty(n, dtype=torch.float32, device=self.device)
              if self.precision in (L.PREC_3XTF32, L.PREC_3XF16) else None)
        L.check(lib.nnab_pack_cqt_bank(dr.data_ptr(), di.data_ptr(), nb, self.width, self.precision, hi.data_ptr(),
                                       L.ptr(lo), L.stream_handle(self.device)), "pack_cqt_bank")
        return schedule, n_ent.value, hi, lo

    def set_bank(self, k_re, k_im, dense: bool = False) -> None:
        lib = L.load()
        kr = np.ascontiguousarray(np.asarray(k_re, dtype=np.float32)) if not torch.is_tensor(k_re) else None
        ki = np.ascontiguousarray(np.asarray(k_im, dtype=np.float32)) if not torch.is_tensor(k_im) else None
        if dense or kr is None:
            sup = np.tile(np.array([0, self.width], dtype=np.int32), (self.n_bins, 1))
        else:
            sup = _row_support(kr, ki)
        dr = torch.as_tensor(k_re).to(self.device, torch.float32).contiguous()
        di = torch.as_tensor(k_im).to(self.device, torch.float32).contiguous()
        self.schedule, self.n_entries, self.packed_hi, self.packed_lo = self._schedule(sup, dr, di)
        self.egemm = self.hybrid = None
        eg_ok = self.hop == 512 and kr is not None and not dense
        if self.method == "hybrid" and eg_ok:  # TF32 or 3xTF32
            span = sup[:, 1] - sup[:, 0]
            n_long = 0
            while n_long < self.n_bins and span[n_long] >= self.LONG_HOPS * self.hop:
                n_long += 1
            eg = self._egemm_tables(sup[:n_long], dr[:n_long], di[:n_long]) if n_long else None
            if eg is not None:
                sch, n_ent, hi, lo = (self._schedule(sup[n_long:], dr[n_long:].contiguous(), di[n_long:].contiguous())
                                      if n_long < self.n_bins else (None, 0, None, None))
                self.hybrid = (eg, sch, n_ent, hi, lo, n_long)
        elif self.method == "egemm" and eg_ok and self.precision == L.PREC_TF32:
            self.egemm = self._egemm_tables(sup, dr, di)

    def _egemm_tables(self, sup, dr, di):
        """Hop-offset GEMM ("E-GEMM", csrc/cqt1992_egemm.cu) tables and packed bank
        for the rows in dr/di; None when the plan does not fit."""
        lib = L.load()
        max_groups = 64
        ct = np.zeros(max_groups * 256, dtype=np.uint16)
        gr = np.zeros(max_groups * 64, dtype=np.int32)
        rt = np.zeros(max_groups * 4 * 65, dtype=np.uint32)
        ng, rm = C.c_int32(), C.c_int32()
        sup = np.ascontiguousarray(sup, dtype=np.int32)
        rc = lib.nnab_cqt_egemm_plan(sup.ctypes.data, int(sup.shape[0]), self.width, self.hop, max_groups,
                                     ct.ctypes.data, gr.ctypes.data, rt.ctypes.data, C.byref(ng), C.byref(rm))
        if rc == L.OK:
            n = ng.value
            col_t = torch.from_numpy(ct[: n * 256].view(np.int16).copy()).to(self.device)
            rows_t = torch.from_numpy(gr[: n * 64].copy()).to(self.device)
            runs_t = torch.from_numpy(rt[: n * 4 * 65].view(np.int32).copy()).to(self.device)
            nb = lib.nnab_cqt_egemm_bank_bytes_prec(n, self.hop, self.precision) // 4
            bank = torch.empty(nb, dtype=torch.float32, device=self.device)
            bank_lo = (torch.empty(nb, dtype=torch.float32, device=self.device)
                       if self.precision in (L.PREC_3XTF32, L.PREC_3XF16) else None)
            L.check(lib.nnab_pack_cqt_egemm(dr.data_ptr(), di.data_ptr(), self.width, self.hop, col_t.data_ptr(),
                                            rows_t.data_ptr(), n, self.precision, bank.data_ptr(), L.ptr(bank_lo),
                                            L.stream_handle(self.device)), "pack_cqt_egemm")
            return (bank, col_t, rows_t, runs_t, n, rm.value, bank_lo)
        return None

    def frames(self, B: int, length: int) -> L.nnab_frames:
        return frames_struct(B, length, self.width, self.hop, self.width // 2, self.pad_mode)

    def n_frames(self, length: int) -> int:
        return geometry(length, self.width, self.hop, self.width // 2, self.pad_mode)[0]

    def forward(self, x: torch.Tensor, kind: str = "magnitude", eps: float = 1e-12) -> torch.Tensor:
        B, length = self.stage(x)
        return self.run_staged(B, length, kind, eps)

    def stage(self, x: torch.Tensor):
        lib = L.load()
        if x.dim() == 1:
            x = x[None]
        if x.device != self.device:
            raise ValueError(f"input on {x.device}, engine on {self.device}")
        x = x.to(torch.float32).contiguous()
        B, length = int(x.shape[0]), int(x.shape[1])
        self.n_frames(length)
        if B:
            f = self.frames(B, length)
            ws = self._ws.get(lib.nnab_stft_workspace_bytes(C.byref(f), self.precision), self.device)
            L.check(lib.nnab_stage_frames(C.byref(f), x.data_ptr(), self.precision, ws.data_ptr(), ws.numel(),
                                          L.stream_handle(self.device)), "stage_frames")
        return B, length

    def run_staged(self, B: int, length: int, kind: str = "magnitude", eps: float = 1e-12) -> torch.Tensor:
        lib = L.load()
        T = self.n_frames(length)
        kinds = {"magnitude": L.OUT_MAGNITUDE, "power": L.OUT_POWER, "complex": L.OUT_COMPLEX,
                 "smooth": L.OUT_SMOOTH_MAG}
        if kind not in kinds:
            raise ValueError(f"output must be one of {sorted(kinds)}, got {kind!r}")
        dt = torch.complex64 if kind == "complex" else torch.float32
        out = torch.empty(B, self.n_bins, T, dtype=dt, device=self.device)
        if B == 0:
            return out
        f = self.frames(B, length)
        ws = self._ws.buf
        if self.hybrid is not None:
            (bank, col_t, rows_t, _, n, rmax, bank_lo), sch, n_ent, s_hi, s_lo, n_long = self.hybrid
            rc = lib.nnab_cqt1992v2_hybrid_staged(C.byref(f), bank.data_ptr(), L.ptr(bank_lo), col_t.data_ptr(),
                                                  rows_t.data_ptr(), n, rmax, L.ptr(s_hi), L.ptr(s_lo),
                                                  L.ptr(sch), n_ent, n_long, self.n_bins, self.precision,
                                                  kinds[kind], float(eps), out.data_ptr(), ws.data_ptr(),
                                                  ws.numel(), L.stream_handle(self.device))
            if rc != L.ENOTSUP:  # ENOTSUP (too few SMs for the E-GEMM pairs): the all-bins schedule below
                L.check(rc, "cqt1992v2_hybrid_staged")
                return out
        if self.egemm is not None:
            bank, col_t, rows_t, runs_t, n, rmax, _ = self.egemm
            rc = lib.nnab_cqt1992v2_egemm_staged(C.byref(f), bank.data_ptr(), col_t.data_ptr(), rows_t.data_ptr(),
                                                 runs_t.data_ptr(), n, rmax, self.n_bins, kinds[kind], float(eps),
                                                 out.data_ptr(),
                                                 ws.data_ptr(), ws.numel(), L.stream_handle(self.device))
            if rc != L.ENOTSUP:
                L.check(rc, "cqt1992v2_egemm_staged")
                return out
        L.check(lib.nnab_cqt1992v2_forward_staged(C.byref(f), self.packed_hi.data_ptr(), L.ptr(self.packed_lo),
                                                  self.n_bins, self.schedule.data_ptr(), self.n_entries,
                                                  self.precision, kinds[kind], float(eps), out.data_ptr(),
                                                  ws.data_ptr(), ws.numel(), L.stream_handle(self.device)),
                "cqt1992v2_forward_staged")
        return out

    def forward_host(self, x_host: torch.Tensor, kind: str = "magnitude", chunk_clips: int = 148,
                     out_host: torch.Tensor | None = None, eps: float = 1e-12) -> torch.Tensor:
        """Pinned host (B, L) -> pinned host (B, n_bins, T), streamed through the
        GPU in chunks with copy/compute overlap (nnab_cqt1992v2_forward_host)."""
        lib = L.load()
        B, length = int(x_host.shape[0]), int(x_host.shape[1])
        T = self.n_frames(length)
        k = {"magnitude": L.OUT_MAGNITUDE, "power": L.OUT_POWER, "complex": L.OUT_COMPLEX}[kind]
        if out_host is None:
            dt = torch.complex64 if kind == "complex" else torch.float32
            out_host = torch.empty(B, self.n_bins, T, dtype=dt, pin_memory=True)
        f = self.frames(B, length)
        ws = self._ws.get(lib.nnab_cqt1992v2_host_scratch_bytes(C.byref(f), self.precision, self.n_bins, k,
                                                                 chunk_clips), self.device)
        if self.hybrid is not None:
            (bank, col_t, rows_t, _, n, rmax, bank_lo), sch, n_ent, s_hi, s_lo, n_long = self.hybrid
            rc = lib.nnab_cqt1992v2_hybrid_forward_host(
                C.byref(f), x_host.data_ptr(), bank.data_ptr(), L.ptr(bank_lo), col_t.data_ptr(), rows_t.data_ptr(),
                n, rmax, L.ptr(s_hi), L.ptr(s_lo), L.ptr(sch), n_ent, n_long, self.n_bins, self.precision, k,
                float(eps), out_host.data_ptr(), int(chunk_clips), ws.data_ptr(), ws.numel(),
                L.stream_handle(self.device))
            if rc != L.ENOTSUP:
                L.check(rc, "cqt1992v2_hybrid_forward_host")
                return out_host
        L.check(lib.nnab_cqt1992v2_forward_host(
            C.byref(f), x_host.data_ptr(), self.packed_hi.data_ptr(), L.ptr(self.packed_lo), self.n_bins,
            self.schedule.data_ptr(), self.n_entries, self.precision, k, float(eps), out_host.data_ptr(),
            int(chunk_clips), ws.data_ptr(), ws.numel(), L.stream_handle(self.device)), "cqt1992v2_forward_host")
        return out_host


class Cqt2010Engine:
    """CQT2010v2's octave recursion (transforms.py:241-323): FIR halvings and
    per-octave short complex convs, all on the device (csrc/cqt2010.cu)."""

    def __init__(self, taps: np.ndarray, top_kernels: np.ndarray, early_stages: int, n_octaves: int,
                 kernel_hop: int, first_bin: int, bins_per_octave: int, n_bins: int, pad_mode: str = "reflect",
                 device="cuda", precision: str = "tf32"):
        self.device = _require_cuda(device)
        # the <= 1e-3 mode is the fused tensor-core chain with FP16 operands under an exact
        # per-clip power-of-two scale ("f16"; "tf32" names the same mode for API symmetry
        # with the other transforms); "fp32" is the FP32 CUDA-core chain (<= 1e-5)
        modes = {"f16": L.PREC_TF32, "tf32": L.PREC_TF32, "fp32": L.PREC_3XTF32, "3xtf32": L.PREC_3XTF32}
        if precision not in modes:
            raise ValueError(f"CQT2010v2 precision must be one of {sorted(modes)}")
        self.precision = modes[precision]
        self.taps = np.ascontiguousarray(np.asarray(taps, dtype=np.float32))
        k = np.asarray(top_kernels)
        self.k_re = torch.from_numpy(np.ascontiguousarray(k.real, dtype=np.float32)).to(self.device)
        self.k_im = torch.from_numpy(np.ascontiguousarray(k.imag, dtype=np.float32)).to(self.device)
        self.n_filters, self.width = int(k.shape[0]), int(k.shape[1])
        self.early_stages, self.n_octaves = int(early_stages), int(n_octaves)
        self.kernel_hop, self.first_bin = int(kernel_hop), int(first_bin)
        self.bins_per_octave, self.n_bins = int(bins_per_octave), int(n_bins)
        if pad_mode not in L.PAD_MODES:
            raise ValueError(f"unknown pad mode {pad_mode!r}")
        self.pad_mode = L.PAD_MODES[pad_mode]
        self._ws = _Workspace()

    def _call(self, x, B, length, kind, out):
        lib = L.load()
        kinds = {"magnitude": L.OUT_MAGNITUDE, "power": L.OUT_POWER, "complex": L.OUT_COMPLEX}
        if kind not in kinds:
            raise ValueError(f"output must be one of {sorted(kinds)}, got {kind!r}")
        need = lib.nnab_cqt2010v2_workspace_bytes(B, length, self.early_stages)
        ws = self._ws.get(need, self.device) if B else None
        T = C.c_int32()
        rc = lib.nnab_cqt2010v2_forward(
            None if x is None else x.data_ptr(), B, length, self.taps.ctypes.data, self.taps.size,
            self.k_re.data_ptr(), self.k_im.data_ptr(), self.n_filters, self.width, self.early_stages,
            self.n_octaves, self.kernel_hop, self.first_bin, self.bins_per_octave, self.n_bins, self.pad_mode,
            kinds[kind], self.precision, None if out is None else out.data_ptr(), C.byref(T),
            None if ws is None else ws.data_ptr(),
            0 if ws is None else ws.numel(), L.stream_handle(self.device))
        return rc, T.value

    def n_frames(self, length: int) -> int:
        lib = L.load()
        T = C.c_int32()
        dummy = torch.empty(1, device=self.device)
        rc = lib.nnab_cqt2010v2_forward(dummy.data_ptr(), 0, length, self.taps.ctypes.data, self.taps.size,
                                        self.k_re.data_ptr(), self.k_im.data_ptr(), self.n_filters, self.width,
                                        self.early_stages, self.n_octaves, self.kernel_hop, self.first_bin,
                                        self.bins_per_octave, self.n_bins, self.pad_mode, L.OUT_MAGNITUDE, self.precision,
                                        dummy.data_ptr(), C.byref(T), None, 0, L.stream_handle(self.device))
        L.check(rc, "cqt2010v2_forward")
        return T.value

    def forward_host(self, x_host: torch.Tensor, kind: str = "magnitude", chunk_clips: int = 148,
                     out_host: torch.Tensor | None = None) -> torch.Tensor:
        """Pinned host (B, L) -> pinned host (B, n_bins, T) through
        nnab_cqt2010v2_forward_host (chunked H2D / compute / D2H overlap)."""
        lib = L.load()
        B, length = int(x_host.shape[0]), int(x_host.shape[1])
        T = self.n_frames(length)
        k = {"magnitude": L.OUT_MAGNITUDE, "power": L.OUT_POWER, "complex": L.OUT_COMPLEX}[kind]
        if out_host is None:
            dt = torch.complex64 if kind == "complex" else torch.float32
            out_host = torch.empty(B, self.n_bins, T, dtype=dt, pin_memory=True)
        ws = self._ws.get(lib.nnab_cqt2010v2_host_scratch_bytes(length, self.early_stages, self.n_bins, T, k,
                                                                 chunk_clips), self.device)
        L.check(lib.nnab_cqt2010v2_forward_host(
            x_host.data_ptr(), B, length, self.taps.ctypes.data, self.taps.size, self.k_re.data_ptr(),
            self.k_im.data_ptr(), self.n_filters, self.width, self.early_stages, self.n_octaves, self.kernel_hop,
            self.first_bin, self.bins_per_octave, self.n_bins, self.pad_mode, k, self.precision,
            out_host.data_ptr(), int(chunk_clips), ws.data_ptr(), ws.numel(), L.stream_handle(self.device)),
            "cqt2010v2_forward_host")
        return out_host

    def forward(self, x: torch.Tensor, kind: str = "magnitude") -> torch.Tensor:
        if x.dim() == 1:
            x = x[None]
        if x.device != self.device:
            raise ValueError(f"input on {x.device}, engine on {self.device}")
        x = x.to(torch.float32).contiguous()
        B, length = int(x.shape[0]), int(x.shape[1])
        T = self.n_frames(length)
        dt = torch.complex64 if kind == "complex" else torch.float32
        out = torch.empty(B, self.n_bins, T, dtype=dt, device=self.device)  # every row is written
        if B == 0:
            return out
        rc, _ = self._call(x, B, length, kind, out)
        L.check(rc, "cqt2010v2_forward")
        return out
