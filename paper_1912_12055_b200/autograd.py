"""Trainable spectrogram layers: forward/backward through the sm_100a kernels.

`DftLayerOp` is the device counterpart of the reference's TrainableLayer +
spectrogram_vjp (gradients.py:28-149) over a whole batch of clips:

  forward   S = sqrt(re^2 + im^2 + eps)           (conv layer, gradients.py:61-67)
            mel = W @ S                           (mel layer,  gradients.py:69-80)
  backward  dW  = g @ S^T                         (gradients.py:118-121)
            dS  = W^T g          (joint mel + trainable STFT, nnAudio trainable_STFT)
            dh  = (dS*re/S, dS*im/S) @ frames     (gradients.py:125-129)
            dx  = overlap-add(coef^T @ h) folded through the pad map (gradients.py:133-149)

Every product is a tcgen05 GEMM (stft_gemm / rgemm); kernel gradients are
summed over all clips of the batch in one reduction (the batch-mean is the
caller's choice of upstream scaling).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib as L
from .engine import DftEngine


def _f32(n_rows: int, n_cols: int, device) -> torch.Tensor:
    return torch.empty(n_rows, n_cols, dtype=torch.float32, device=device)


class DftLayerOp:
    """Batched forward/backward for a DFT-type bank (STFT or time-domain CQT
    rows) with an optional Mel projection on top."""

    def __init__(self, h_re, h_im, hop: int, center: bool = True, pad_mode: str = "reflect", eps: float = 1e-12,
                 precision: str = "tf32", device="cuda", phasor: str = "split"):
        # the Nyquist cosine row rides in bin 0's sine slot while both zero sine rows stay exactly
        # zero (8 bank tiles instead of 9 for n_fft = 2048); re-checked at every set_bank
        self.engine = DftEngine(h_re, h_im, hop, center, pad_mode, precision=precision, device=device,
                                allow_fold="exact", f16_ok=False)
        self.eps = float(eps)
        self.device = self.engine.device
        self.prec = self.engine.precision
        self.split = self.prec == L.PREC_3XTF32
        self.reducer = None  # dist.GradReducer while armed: gradient blocks are all-reduced as they finish
        # TF32 mode: every frame's gradient is weighted by the unit phasor (re/S, im/S),
        # whose direction a one-pass forward gets wrong where |X| is near zero (the
        # rounding error of re, im divided by S).  phasor="split" computes the
        # forward in a split mode (3xF16, or 3xTF32 when the FP16 staging would lay
        # the frames out differently) and saves the FP32-accurate phasor, keeping the
        # backward GEMMs TF32; phasor="tf32" is the one-pass forward (faster, with
        # that gradient tail).
        if phasor not in ("split", "tf32"):
            raise ValueError("phasor must be 'split' or 'tf32'")
        # The 3xTF32 mode's forward runs 3xF16 where it stages the same rows (half the
        # operand error of 3xTF32, 2.8e-6 vs 5e-6, and the same phasor argument one level down).
        self.fwd_engine = None
        eng = self.engine
        same_rows = self._f16_same_rows(eng.n_fft, eng.hop)
        if (self.prec == L.PREC_TF32 and phasor == "split") or (self.split and same_rows):
            self.fwd_prec = L.PREC_3XF16 if same_rows else L.PREC_3XTF32
            self.fwd_engine = DftEngine(h_re, h_im, hop, center, pad_mode, precision="3xf16", device=device,
                                        allow_fold="exact")
            if self.fwd_prec == L.PREC_3XTF32:
                self.fwd_engine.precision = L.PREC_3XTF32
                self.fwd_engine.set_bank(h_re, h_im)
        elif (self.prec == L.PREC_TF32 and same_rows and eng.hop % 64 == 0
              and os.environ.get("NNAB_F16_DK", "1") != "0"):
            # phasor="tf32" (one-pass forward): FP16 operands keep TF32's 11 bits at twice the rate,
            # and their staging feeds the one-pass FP16 kernel gradient
            self.fwd_prec = L.PREC_F16
            self.fwd_engine = DftEngine(h_re, h_im, hop, center, pad_mode, precision="f16", device=device,
                                        allow_fold="exact")
        # the kernel gradient runs on FP16 tensor cores over the 3xF16 forward's staging
        # (nnab_kernel_grad_f16) where that staging holds hop rows of 64-sample multiples:
        # 3xF16 in FP32 mode, one FP16 pass (11-bit operands, as TF32) in TF32 mode
        hop, k64 = eng.hop, (eng.n_fft + 63) // 64 * 64
        self.f16_dk = (self.fwd_engine is not None and self.fwd_prec in (L.PREC_3XF16, L.PREC_F16)
                       and hop % 64 == 0 and hop <= k64 and os.environ.get("NNAB_F16_DK", "1") != "0")

    @staticmethod
    def _f16_same_rows(n_fft: int, hop: int) -> bool:
        """True when the FP16 staging (64-sample K blocks) has the TF32 staging's rows per clip."""
        k32, k64 = (n_fft + 31) // 32 * 32, (n_fft + 63) // 64 * 64
        hr32, hr64 = hop % 32 == 0 and hop <= k32, hop % 64 == 0 and hop <= k64
        if hr32 != hr64:
            return False
        return not hr32 or (k32 + hop - 1) // hop == (k64 + hop - 1) // hop

    @property
    def n_bins(self):
        return self.engine.n_bins

    def set_bank(self, h_re: torch.Tensor, h_im: torch.Tensor):
        self.engine.set_bank(h_re.detach(), h_im.detach())
        if self.fwd_engine is not None:
            self.fwd_engine.set_bank(h_re.detach(), h_im.detach())

    # ------------------------------------------------------------ forward
    def forward(self, x: torch.Tensor, mel_w: torch.Tensor | None = None, phasor_grads: bool = True):
        """x (B, L) -> (S (B, F, T) or mel (B, n_mels, T), saved state).
        phasor_grads=False (only the mel weights need a gradient): the one-pass
        forward, whose |X| is all dW needs."""
        lib, eng = L.load(), self.engine
        if x.dim() == 1:
            x = x[None]
        x = x.detach().to(self.device, torch.float32).contiguous()
        B, length = int(x.shape[0]), int(x.shape[1])
        T = eng.n_frames(length)
        f = eng.frames(B, length)
        stream = L.stream_handle(self.device)
        fe = self.fwd_engine if (phasor_grads or self.split) else None
        if fe is not None and (self.fwd_prec == L.PREC_3XTF32 or self.f16_dk):
            ws = None  # one staging: the forward's rows are the frames the dK GEMM reads
        else:
            ws = torch.empty(lib.nnab_stft_workspace_bytes(C.byref(f), self.prec), dtype=torch.uint8,
                             device=self.device)
            L.check(lib.nnab_stage_frames(C.byref(f), x.data_ptr(), self.prec, ws.data_ptr(), ws.numel(), stream),
                    "stage_frames")
        if fe is not None:
            ws_f = torch.empty(lib.nnab_stft_workspace_bytes(C.byref(f), self.fwd_prec), dtype=torch.uint8,
                               device=self.device)
            L.check(lib.nnab_stage_frames(C.byref(f), x.data_ptr(), self.fwd_prec, ws_f.data_ptr(), ws_f.numel(),
                                          stream), "stage_frames")
            if ws is None:
                ws = ws_f
        ld = lib.nnab_slots_ld(C.byref(f))
        F = self.n_bins
        R = self._rows_per_clip(length)
        # TF32: the backward only needs the unit phasor (re/S, im/S), saved as FP16
        # pairs in one 32-bit word per (bin, slot); 3xTF32 keeps re and im in FP32
        re_s = _f32(F, ld, self.device)
        im_s = _f32(F, ld, self.device) if self.split else None
        # split modes: |X| saved as its 3xTF32 (hi, lo) pair [2][F][ld] straight from the epilogue
        mag_split = mel_w is not None and fe is not None and self.split
        mag_s = _f32((2 if mag_split else 1) * F, ld, self.device) if mel_w is not None else None
        # mel layer: the STFT GEMM only saves re/im/S per slot; W @ S then runs as a
        # tcgen05 GEMM (a trained W is dense, so the epilogue's banded CUDA-core path
        # would be latency-bound)
        out = None if mel_w is not None else torch.empty(B, F, T, device=self.device)
        if fe is not None:  # split forward; TF32 mode: TF32-backward saves (FP32-accurate phasor)
            flag = (L.SAVE_MAG_SPLIT if mag_split else 0) if self.split else L.SAVE_PHASOR
            L.check(lib.nnab_stft_forward_train_staged(
                C.byref(f), fe.packed_hi.data_ptr(), L.ptr(fe.packed_lo), F, fe.fold, self.fwd_prec,
                L.OUT_SMOOTH_MAG | flag, 1.0, self.eps, None, 0, 0, None, L.ptr(out), re_s.data_ptr(), L.ptr(im_s),
                L.ptr(mag_s), ld, ws_f.data_ptr(), ws_f.numel(), stream), "stft_forward_train")
        else:
            L.check(lib.nnab_stft_forward_train_staged(
                C.byref(f), eng.packed_hi.data_ptr(), L.ptr(eng.packed_lo), F, eng.fold, self.prec, L.OUT_SMOOTH_MAG,
                1.0, self.eps, None, 0, 0, None, L.ptr(out), re_s.data_ptr(), L.ptr(im_s), L.ptr(mag_s), ld,
                ws.data_ptr(), ws.numel(), stream), "stft_forward_train")
        saved = {"ws": ws, "re": re_s, "im": im_s, "mag": mag_s, "B": B, "L": length, "T": T, "ld": ld, "R": R}
        if mel_w is not None:
            nm = int(mel_w.shape[0])
            kp = (F + 31) // 32 * 32
            wp = torch.zeros(nm, kp, device=self.device)
            wp[:, :F] = mel_w.detach().to(self.device, torch.float32)
            if mag_split:
                magp = (mag_s[:F], mag_s[F:])
            else:
                magp = self._split(mag_s) if self.split else (mag_s, None)
            saved["magp"] = magp
            out = torch.empty(B, nm, T, device=self.device)
            wsp = self._split(wp)
            if R % 4 == 0 and kp <= 2048:  # W @ S straight into (B, n_mels, T)
                L.check(lib.nnab_mel_forward_slots(nm, ld, kp, wsp[0].data_ptr(), L.ptr(wsp[1]), magp[0].data_ptr(),
                                                   L.ptr(magp[1]), F, B, R, T, self.prec, out.data_ptr(), stream),
                        "mel_forward_slots")
            else:
                mel_s = _f32(nm, ld, self.device)
                self._rgemm(nm, ld, kp, wsp, kp, magp, ld, 1, ld, F, mel_s, ld)
                L.check(lib.nnab_from_slots(mel_s.data_ptr(), B, nm, T, R, ld, out.data_ptr(), stream), "from_slots")
        return out, saved

    def _rows_per_clip(self, length):
        from .engine import geometry
        pad = self.engine.n_fft // 2 if self.engine.center else 0
        return geometry(length, self.engine.n_fft, self.engine.hop, pad, self.engine.pad_mode)[2]

    # ------------------------------------------------------------ helpers
    def _split(self, t: torch.Tensor):
        lib = L.load()
        hi = torch.empty_like(t)
        lo = torch.empty_like(t) if self.split else None
        L.check(lib.nnab_tf32_split(t.data_ptr(), t.numel(), self.prec, hi.data_ptr(), L.ptr(lo),
                                    L.stream_handle(self.device)), "tf32_split")
        return hi, lo

    def _rgemm(self, M, N, K, a, lda, b, ldb, b_mn, b_row_len, b_rows, c, ldc, splits=0):
        lib = L.load()
        part_bytes = lib.nnab_rgemm_partial_bytes(M, N, K, splits)
        part = torch.empty(max(part_bytes // 4, 1), dtype=torch.float32, device=self.device)
        L.check(lib.nnab_rgemm(M, N, K, a[0].data_ptr(), L.ptr(a[1]), lda, b[0].data_ptr(), L.ptr(b[1]), ldb, b_mn,
                               b_row_len, b_rows, c.data_ptr(), ldc, splits, part.data_ptr(), self.prec,
                               L.stream_handle(self.device)), "rgemm")

    def _f16_operands(self, F, ld):
        """FP16 hi/lo coef [2F][ld] and the int32 row exponents [2F + 1] of the 3xF16 dK"""
        c16 = tuple(torch.empty(2 * F, ld, dtype=torch.float16, device=self.device) if i == 0 or self.split
                    else None for i in range(2))
        return c16, torch.empty(2 * F + 1, dtype=torch.int32, device=self.device)

    # ------------------------------------------------------------ backward
    def backward(self, saved: dict, g: torch.Tensor, h_re=None, h_im=None, mel_w: torch.Tensor | None = None,
                 need_bank: bool = True, need_mel: bool = False, need_x: bool = False):
        """g: upstream grad of the forward output.  Returns dict with any of
        'h_re', 'h_im' (F, n_fft), 'weights' (n_mels, F), 'x' (B, L)."""
        lib, eng = L.load(), self.engine
        stream = L.stream_handle(self.device)
        g = g.detach().to(self.device, torch.float32).contiguous()
        B, T, ld, R, length = saved["B"], saved["T"], saved["ld"], saved["R"], saved["L"]
        F, n_fft = self.n_bins, eng.n_fft
        f = eng.frames(B, length)
        grads = {}
        ds = None
        use16 = self.f16_dk and need_bank
        if mel_w is not None:
            nm = int(mel_w.shape[0])
            gsp = (_f32(nm, ld, self.device), _f32(nm, ld, self.device) if self.split else None)
            L.check(lib.nnab_grad_to_slots_split(g.data_ptr(), B, nm, T, R, ld, self.prec, gsp[0].data_ptr(),
                                                 L.ptr(gsp[1]), stream), "grad_to_slots_split")
            if need_mel:  # dW[m][f] = sum_slot g[m][slot] S[f][slot]
                magp = saved["magp"]
                dW = torch.empty(nm, F, device=self.device)
                self._rgemm(nm, F, ld, gsp, ld, magp, ld, 0, 0, 0, dW, F)
                grads["weights"] = dW
                if self.reducer is not None:  # overlaps the coef and dK GEMMs below
                    self.reducer.launch(dW)
            if need_bank or need_x:  # dS[f][slot] = sum_m W[m][f] g[m][slot]
                kp = (nm + 31) // 32 * 32
                wt_hi = _f32(F, kp, self.device)
                wt_lo = _f32(F, kp, self.device) if self.split else None
                L.check(lib.nnab_transpose_pad(mel_w.detach().float().contiguous().data_ptr(), nm, F, kp, self.prec,
                                               wt_hi.data_ptr(), L.ptr(wt_lo), stream), "transpose_pad")
                # coef = (dS*re/S, dS*im/S) straight from the dS GEMM's epilogue
                if use16:  # the 3xF16 dK operand
                    c16, rexp = self._f16_operands(F, ld)
                    L.check(lib.nnab_mel_dft_coef_f16(
                        C.byref(f), saved["ws"].data_ptr(), saved["ws"].numel(), self.fwd_prec, F, ld, kp,
                        wt_hi.data_ptr(),
                        L.ptr(wt_lo), gsp[0].data_ptr(), L.ptr(gsp[1]), nm, saved["re"].data_ptr(),
                        L.ptr(saved["im"]), self.eps, c16[0].data_ptr(), L.ptr(c16[1]), rexp.data_ptr(),
                        stream), "mel_dft_coef_f16")
                if need_x or not use16:
                    coef_hi = _f32(2 * F, ld, self.device)
                    coef_lo = _f32(2 * F, ld, self.device) if self.split else None
                    L.check(lib.nnab_mel_dft_coef(F, ld, kp, wt_hi.data_ptr(), L.ptr(wt_lo), gsp[0].data_ptr(),
                                                  L.ptr(gsp[1]), nm, saved["re"].data_ptr(), L.ptr(saved["im"]),
                                                  self.eps, self.prec, coef_hi.data_ptr(), L.ptr(coef_lo), stream),
                            "mel_dft_coef")
                ds = True
        if not (need_bank or need_x):
            if self.reducer is not None:
                self.reducer.wait()
            return grads
        if ds is None and (need_x or not use16):
            coef_hi = _f32(2 * F, ld, self.device)
            coef_lo = _f32(2 * F, ld, self.device) if self.split else None
            L.check(lib.nnab_dft_coef(None, g.data_ptr(), saved["re"].data_ptr(), L.ptr(saved["im"]), F, B, T,
                                      R, ld, self.eps, self.prec, coef_hi.data_ptr(), L.ptr(coef_lo), stream),
                    "dft_coef")
        ws = saved["ws"]
        if use16 and ds is None:  # conv layer: coef from g directly
            c16, rexp = self._f16_operands(F, ld)
            L.check(lib.nnab_dft_coef_f16(C.byref(f), ws.data_ptr(), ws.numel(), self.fwd_prec, g.data_ptr(),
                                          saved["re"].data_ptr(),
                                          L.ptr(saved["im"]), F, T, ld, self.eps, c16[0].data_ptr(),
                                          L.ptr(c16[1]), rexp.data_ptr(), stream), "dft_coef_f16")
        if need_bank and use16:
            dk = _f32(2 * F, n_fft, self.device)
            blocks = [(0, 2 * F)] if self.reducer is None or 2 * F <= 1280 else [(0, 1024), (1024, 2 * F)]
            for r0, r1 in blocks:
                part = torch.empty(max(lib.nnab_rgemm_partial_bytes(r1 - r0, n_fft, ld, 0) // 4, 1),
                                   device=self.device)
                L.check(lib.nnab_kernel_grad_f16(C.byref(f), c16[0].data_ptr() + 2 * r0 * ld,
                                                 None if c16[1] is None else c16[1].data_ptr() + 2 * r0 * ld,
                                                 r1 - r0, ld,
                                                 rexp.data_ptr() + 4 * r0, dk.data_ptr() + 4 * r0 * n_fft, n_fft,
                                                 ws.data_ptr(), ws.numel(), self.fwd_prec, part.data_ptr(), 0,
                                                 stream),
                        "kernel_grad_f16")
                if self.reducer is not None:
                    self.reducer.launch(dk[r0:r1])
            grads["h_re"], grads["h_im"] = dk[:F], dk[F:]
        elif need_bank:
            dk = _f32(2 * F, n_fft, self.device)
            # with a reducer: rows [0, 1024) first (whole 256-row tiles), all-reduced while
            # the remaining rows' GEMM runs; without: one launch over all 2F rows
            blocks = [(0, 2 * F)] if self.reducer is None or 2 * F <= 1280 else [(0, 1024), (1024, 2 * F)]
            for r0, r1 in blocks:
                part = torch.empty(max(lib.nnab_rgemm_partial_bytes(r1 - r0, n_fft, ld, 0) // 4, 1),
                                   device=self.device)
                L.check(lib.nnab_kernel_grad(C.byref(f), coef_hi.data_ptr() + 4 * r0 * ld,
                                             None if coef_lo is None else coef_lo.data_ptr() + 4 * r0 * ld,
                                             r1 - r0, ld, self.prec, dk.data_ptr() + 4 * r0 * n_fft, n_fft,
                                             ws.data_ptr(), ws.numel(), part.data_ptr(), 0, stream), "kernel_grad")
                if self.reducer is not None:
                    self.reducer.launch(dk[r0:r1])
            grads["h_re"], grads["h_im"] = dk[:F], dk[F:]
        if need_x:  # frame grads^T [tap][slot] = h^T @ coef, then overlap-add + pad fold
            h = torch.cat([torch.as_tensor(h_re), torch.as_tensor(h_im)]).to(self.device, torch.float32).contiguous()
            kp = (2 * F + 31) // 32 * 32
            ht_hi = _f32(n_fft, kp, self.device)
            ht_lo = _f32(n_fft, kp, self.device) if self.split else None
            L.check(lib.nnab_transpose_pad(h.data_ptr(), 2 * F, n_fft, kp, self.prec, ht_hi.data_ptr(),
                                           L.ptr(ht_lo), stream), "transpose_pad")
            fgt = _f32(n_fft, ld, self.device)
            self._rgemm(n_fft, ld, kp, (ht_hi, ht_lo), kp, (coef_hi, coef_lo), ld, 1, ld, 2 * F, fgt, ld)
            gx = torch.empty(B, length, device=self.device)
            L.check(lib.nnab_input_grad(C.byref(f), fgt.data_ptr(), ld, gx.data_ptr(), stream), "input_grad")
            grads["x"] = gx
        if self.reducer is not None:  # order the compute stream after every reduction
            self.reducer.wait()
        return grads


class DftLayerFunction(torch.autograd.Function):
    """autograd wrapper: out = layer(x; h_re, h_im[, W])."""

    @staticmethod
    def forward(ctx, x, h_re, h_im, mel_w, op: DftLayerOp, bank_version: int):
        if op._bank_version != bank_version:
            op.set_bank(h_re, h_im)
            op._bank_version = bank_version
        nig = ctx.needs_input_grad
        out, saved = op.forward(x, mel_w, phasor_grads=bool(nig[0] or nig[1] or nig[2]))
        ctx.op, ctx.saved = op, saved
        ctx.save_for_backward(h_re, h_im, mel_w if mel_w is not None else torch.empty(0))
        ctx.has_mel = mel_w is not None
        return out

    @staticmethod
    def backward(ctx, g):
        h_re, h_im, mel_w = ctx.saved_tensors
        need_x, need_bank = ctx.needs_input_grad[0], ctx.needs_input_grad[1] or ctx.needs_input_grad[2]
        need_mel = ctx.has_mel and ctx.needs_input_grad[3]
        if need_x and ctx.has_mel:
            raise NotImplementedError("input gradients are only provided for convolution layers")  # gradients.py:122-123
        gr = ctx.op.backward(ctx.saved, g, h_re, h_im, mel_w if ctx.has_mel else None, need_bank=need_bank,
                             need_mel=need_mel, need_x=need_x)
        ctx.saved = None
        return (gr.get("x"), gr.get("h_re"), gr.get("h_im"), gr.get("weights") if ctx.has_mel else None, None, None)
