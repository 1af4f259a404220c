"""ctypes binding of libnnab.so (the C ABI declared in include/nnab.h).

The library is built in-tree by `make` (or `__graft_entry__.build()`).  There
is no fallback: if the library or an sm_100 device is missing, every call
raises, so a run can never silently measure a CPU path.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NNAB_LIB") or os.path.join(_HERE, "libnnab.so")  # NNAB_LIB: debug builds

OK, EINVAL, ECUDA, ENOTSUP, ENODEV = 0, 1, 2, 3, 4
PAD_REFLECT, PAD_ZERO = 0, 1
OUT_MAGNITUDE, OUT_POWER, OUT_COMPLEX, OUT_MEL, OUT_SMOOTH_MAG = 0, 1, 2, 3, 4
OUT_LOG = 0x100  # flag: log(value + eps) in the fused epilogue (STFT / Mel)
SAVE_MAG_SPLIT = 0x400  # flag (training forward, split modes): |X| saved as the 3xTF32 hi / lo pair
SAVE_PHASOR = 0x200  # flag (training forward): TF32-backward saves from a split-precision forward
PREC_TF32, PREC_3XTF32, PREC_F16, PREC_3XF16 = 0, 1, 2, 3
PAD_MODES = {"reflect": PAD_REFLECT, "constant_zero": PAD_ZERO, "constant": PAD_ZERO}
# precision names -> operand modes.  "tf32" / "f16": one pass, peak-normalised error
# <= 1e-3 (FP16 operands under exact power-of-two scales: TF32's 11-bit significand at
# twice the tensor rate).  "fp32": <= 1e-5 (3xTF32; the STFT / Mel engine runs it as
# 3xF16, the same accuracy at half the tensor-core time).
PRECISIONS = {"tf32": PREC_TF32, "fp32": PREC_3XTF32, "3xtf32": PREC_3XTF32, "f16": PREC_F16, "3xf16": PREC_3XF16}


class NnabError(RuntimeError):
    """A libnnab call failed (CUDA error, unsupported configuration, no device)."""


class nnab_frames(C.Structure):
    _fields_ = [("batch", C.c_int64), ("length", C.c_int64), ("width", C.c_int32), ("hop", C.c_int32),
                ("pad", C.c_int32), ("pad_mode", C.c_int32)]


_vp, _fp, _ip, _i32, _i64, _f32, _sz = C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_size_t
_FR = C.POINTER(nnab_frames)

# name -> (restype, argtypes); every symbol include/nnab.h declares.
SIGNATURES = {
    "nnab_version": (C.c_int, []),
    "nnab_strerror": (C.c_char_p, [C.c_int]),
    "nnab_last_error": (C.c_char_p, []),
    "nnab_launch_count": (C.c_uint64, []),
    "nnab_frames_geometry": (C.c_int, [_FR, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "nnab_dft_bank_tiles": (C.c_int, [_i32, _i32]),
    "nnab_dft_bank_bytes": (_sz, [_i32, _i32, _i32]),
    "nnab_dft_bank_bytes_prec": (_sz, [_i32, _i32, _i32, _i32]),
    "nnab_pack_dft_bank": (C.c_int, [_fp, _fp, _i32, _i32, _i32, _i32, _fp, _fp, _vp]),
    "nnab_stft_workspace_bytes": (_sz, [_FR, _i32]),
    "nnab_stft_forward": (C.c_int, [_FR, _fp, _fp, _fp, _i32, _i32, _i32, _i32, _f32, _f32, _fp, _i32, _i32, _ip,
                                    _fp, _vp, _sz, _vp]),
    "nnab_stage_frames": (C.c_int, [_FR, _fp, _i32, _vp, _sz, _vp]),
    "nnab_stft_forward_staged": (C.c_int, [_FR, _fp, _fp, _i32, _i32, _i32, _i32, _f32, _f32, _fp, _i32, _i32,
                                           _ip, _fp, _vp, _sz, _vp]),
    "nnab_cqt1992v2_forward_staged": (C.c_int, [_FR, _fp, _fp, _i32, _ip, _i32, _i32, _i32, _f32, _fp, _vp, _sz,
                                                _vp]),
    "nnab_stft_host_scratch_bytes": (_sz, [_FR, _i32, _i32, _i64]),
    "nnab_stft_forward_host": (C.c_int, [_FR, _fp, _fp, _fp, _i32, _i32, _i32, _i32, _f32, _f32, _fp, _i32, _i32,
                                         _ip, _fp, _i64, _vp, _sz, _vp]),
    "nnab_slots_ld": (_i64, [_FR]),
    "nnab_stft_forward_train_staged": (C.c_int, [_FR, _fp, _fp, _i32, _i32, _i32, _i32, _f32, _f32, _fp, _i32, _i32,
                                                 _ip, _fp, _fp, _fp, _fp, _i64, _vp, _sz, _vp]),
    "nnab_grad_to_slots": (C.c_int, [_fp, _i64, _i32, _i32, _i32, _i64, _fp, _vp]),
    "nnab_grad_to_slots_split": (C.c_int, [_fp, _i64, _i32, _i32, _i32, _i64, _i32, _fp, _fp, _vp]),
    "nnab_from_slots": (C.c_int, [_fp, _i64, _i32, _i32, _i32, _i64, _fp, _vp]),
    "nnab_dft_coef": (C.c_int, [_fp, _fp, _fp, _fp, _i32, _i64, _i32, _i32, _i64, _f32, _i32, _fp, _fp, _vp]),
    "nnab_mel_forward_slots": (C.c_int, [_i32, _i64, _i32, _fp, _fp, _fp, _fp, _i32, _i64, _i32, _i32, _i32, _fp, _vp]),
    "nnab_mel_dft_coef": (C.c_int, [_i32, _i64, _i32, _fp, _fp, _fp, _fp, _i32, _fp, _fp, _f32, _i32, _fp, _fp, _vp]),
    "nnab_transpose_pad": (C.c_int, [_fp, _i32, _i32, _i32, _i32, _fp, _fp, _vp]),
    "nnab_tf32_split": (C.c_int, [_fp, _i64, _i32, _fp, _fp, _vp]),
    "nnab_rgemm_partial_bytes": (_sz, [_i32, _i32, _i64, _i32]),
    "nnab_rgemm": (C.c_int, [_i32, _i32, _i64, _fp, _fp, _i64, _fp, _fp, _i64, _i32, _i32, _i64, _fp, _i64, _i32,
                             _fp, _i32, _vp]),
    "nnab_kernel_grad": (C.c_int, [_FR, _fp, _fp, _i32, _i64, _i32, _fp, _i64, _vp, _sz, _fp, _i32, _vp]),
    "nnab_input_grad": (C.c_int, [_FR, _fp, _i64, _fp, _vp]),
    "nnab_mel_dft_coef_f16": (C.c_int, [_FR, _vp, _sz, _i32, _i32, _i64, _i32, _fp, _fp, _fp, _fp, _i32, _fp, _fp, _f32,
                                        _vp, _vp, _ip, _vp]),
    "nnab_dft_coef_f16": (C.c_int, [_FR, _vp, _sz, _i32, _fp, _fp, _fp, _i32, _i32, _i64, _f32, _vp, _vp, _ip, _vp]),
    "nnab_kernel_grad_f16": (C.c_int, [_FR, _vp, _vp, _i32, _i64, _ip, _fp, _i64, _vp, _sz, _i32, _fp, _i32, _vp]),
    "nnab_cqt_bank_tiles": (C.c_int, [_i32]),
    "nnab_cqt_bank_bytes": (_sz, [_i32, _i32]),
    "nnab_cqt_bank_bytes_prec": (_sz, [_i32, _i32, _i32]),
    "nnab_cqt_egemm_bank_bytes_prec": (_sz, [_i32, _i32, _i32]),
    "nnab_pack_cqt_bank": (C.c_int, [_fp, _fp, _i32, _i32, _i32, _fp, _fp, _vp]),
    "nnab_cqt_schedule": (C.c_int, [_ip, _i32, _i32, _i32, _ip, C.POINTER(_i32)]),
    "nnab_cqt1992v2_forward": (C.c_int, [_FR, _fp, _fp, _fp, _i32, _ip, _i32, _i32, _i32, _f32, _fp, _vp, _sz,
                                         _vp]),
    "nnab_cqt_egemm_plan": (C.c_int, [_ip, _i32, _i32, _i32, _i32, _vp, _ip, _vp, C.POINTER(_i32),
                                      C.POINTER(_i32)]),
    "nnab_cqt_egemm_bank_bytes": (_sz, [_i32, _i32]),
    "nnab_pack_cqt_egemm": (C.c_int, [_fp, _fp, _i32, _i32, _vp, _ip, _i32, _i32, _fp, _fp, _vp]),
    "nnab_cqt1992v2_egemm_staged": (C.c_int, [_FR, _fp, _vp, _ip, _vp, _i32, _i32, _i32, _i32, _f32, _fp, _vp,
                                              _sz, _vp]),
    "nnab_cqt1992v2_hybrid_staged": (C.c_int, [_FR, _fp, _fp, _vp, _ip, _i32, _i32, _fp, _fp, _ip, _i32, _i32, _i32,
                                               _i32, _i32, _f32, _fp, _vp, _sz, _vp]),
    "nnab_cqt1992v2_hybrid_forward": (C.c_int, [_FR, _fp, _fp, _fp, _vp, _ip, _i32, _i32, _fp, _fp, _ip, _i32,
                                                _i32, _i32, _i32, _i32, _f32, _fp, _vp, _sz, _vp]),
    "nnab_cqt1992v2_hybrid_forward_host": (C.c_int, [_FR, _fp, _fp, _fp, _vp, _ip, _i32, _i32, _fp, _fp, _ip,
                                                     _i32, _i32, _i32, _i32, _i32, _f32, _fp, _i64, _vp, _sz, _vp]),
    "nnab_cqt1992v2_host_scratch_bytes": (_sz, [_FR, _i32, _i32, _i32, _i64]),
    "nnab_cqt1992v2_forward_host": (C.c_int, [_FR, _fp, _fp, _fp, _i32, _ip, _i32, _i32, _i32, _f32, _fp, _i64,
                                              _vp, _sz, _vp]),
    "nnab_layer_vjp_workspace_bytes": (_sz, [_FR, _i32, _i32, _i32, _i32]),
    "nnab_layer_vjp": (C.c_int, [_FR, _fp, _fp, _fp, _i32, _fp, _fp, _fp, _i32, _fp, _f32, _i32, _fp, _fp, _fp, _vp,
                                 _sz, _vp]),
    "nnab_pad_signal": (C.c_int, [_fp, _i64, _i64, _i64, _i64, _i32, _fp, _vp]),
    "nnab_downsample2": (C.c_int, [_fp, _i64, _i64, _fp, _i32, _fp, _vp]),
    "nnab_decode_wav": (C.c_int, [_vp, _i64, _i32, _i32, _fp, _vp]),
    "nnab_widen_f64": (C.c_int, [_fp, _i64, _vp, _vp]),
    "nnab_cqt2010v2_workspace_bytes": (_sz, [_i64, _i64, _i32]),
    "nnab_cqt2010v2_host_scratch_bytes": (_sz, [_i64, _i32, _i32, _i32, _i32, _i64]),
    "nnab_cqt2010v2_forward_host": (C.c_int, [_fp, _i64, _i64, _fp, _i32, _fp, _fp, _i32, _i32, _i32, _i32, _i32,
                                              _i32, _i32, _i32, _i32, _i32, _i32, _fp, _i64, _vp, _sz, _vp]),
    "nnab_cqt2010v2_forward": (C.c_int, [_fp, _i64, _i64, _fp, _i32, _fp, _fp, _i32, _i32, _i32, _i32, _i32, _i32,
                                         _i32, _i32, _i32, _i32, _i32, _fp, C.POINTER(_i32), _vp, _sz, _vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load libnnab.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NnabError(f"{LIB_PATH} is missing: build it with `make` (the CUDA path has no fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == OK:
        return
    lib = load()
    msg = lib.nnab_strerror(rc).decode()
    detail = lib.nnab_last_error().decode()
    if rc == EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise NnabError(f"{what}: {msg}" + (f" ({detail})" if detail else ""))


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
