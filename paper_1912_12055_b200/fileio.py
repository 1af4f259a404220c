"""File formats either side of the hot path,
with the reference's names, layouts and errors:

  read_wav(path)             wavio.py:19-68   -> spectro.Signal on the device
  read_wav_batch(paths)      same, equal-length files -> (B, L) CUDA tensor
  write_spec(path, spec)     specfile.py:26-43 (byte-identical files)
  read_spec(path)            specfile.py:46-72

The RIFF / NASP headers are parsed on the host (a few dozen bytes); the WAV
data chunk crosses PCIe as raw bytes (PCM16: half the bytes of float32) and is
decoded, scaled and mono-mixed by one kernel (csrc/io.cu); SpecFile payloads
are widened to float64 on the device.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _lib as L
from .engine import _require_cuda
from .spectro import Signal, Spectrogram

_FORMAT_PCM = 1
_FORMAT_IEEE_FLOAT = 3
_MAGIC = b"NASP"
_VERSION = 1
_HEADER = struct.Struct("<4sIBBHIIdI")
_DTYPE_CODES = {"f32": 0, "f64": 1}
_KIND_CODES = {"magnitude": 0, "power": 1, "complex": 2}
_KIND_NAMES = {v: k for k, v in _KIND_CODES.items()}


class CorruptFileError(ValueError):
    """errors.py: the file's container structure is damaged or inconsistent."""


class UnsupportedFormatError(ValueError):
    """errors.py: the file uses a codec or layout this library does not read."""


def _parse_wav(path):
    """wavio.py:26-63 -- RIFF chunk walk and format checks; returns
    (payload bytes of whole frames, channels, format tag, sample rate)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < 12 or data[:4] != b"RIFF" or data[8:12] != b"WAVE":
        raise CorruptFileError(f"{path}: not a RIFF/WAVE file")
    fmt = None
    payload = None
    pos = 12
    while pos + 8 <= len(data):
        chunk_id = data[pos:pos + 4]
        (size,) = struct.unpack_from("<I", data, pos + 4)
        body = data[pos + 8:pos + 8 + size]
        if len(body) < size:
            raise CorruptFileError(f"{path}: truncated {chunk_id!r} chunk")
        if chunk_id == b"fmt ":
            if size < 16:
                raise CorruptFileError(f"{path}: fmt chunk too short")
            fmt = struct.unpack_from("<HHIIHH", body, 0)
        elif chunk_id == b"data":
            payload = body
        pos += 8 + size + (size & 1)
    if fmt is None or payload is None:
        raise CorruptFileError(f"{path}: missing fmt or data chunk")
    audio_format, channels, sample_rate, _, _, bits = fmt
    if channels < 1:
        raise CorruptFileError(f"{path}: invalid channel count {channels}")
    if audio_format == _FORMAT_PCM and bits == 16:
        width = 2
    elif audio_format == _FORMAT_IEEE_FLOAT and bits == 32:
        width = 4
    else:
        raise UnsupportedFormatError(
            f"{path}: unsupported encoding (format tag {audio_format}, {bits}-bit); "
            "only PCM 16-bit and IEEE float 32-bit are readable")
    n_frames = (len(payload) // width) // channels
    return payload[: n_frames * channels * width], channels, audio_format, float(sample_rate), n_frames


def _decode_into(payload: bytes, channels: int, fmt: int, n_frames: int, out: torch.Tensor, device) -> None:
    raw = torch.frombuffer(bytearray(payload), dtype=torch.uint8) if payload else torch.empty(0, dtype=torch.uint8)
    dev_raw = raw.pin_memory().to(device, non_blocking=True) if raw.numel() else None
    if n_frames:
        L.check(L.load().nnab_decode_wav(dev_raw.data_ptr(), n_frames, channels, fmt, out.data_ptr(),
                                         L.stream_handle(device)), "decode_wav")


def read_wav(path, device="cuda") -> Signal:
    """wavio.py:19-68 -- PCM16 / float32 WAV, any channel count, averaged to
    mono; decoded on the device."""
    dev = _require_cuda(device)
    payload, channels, fmt, sr, n = _parse_wav(path)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    _decode_into(payload, channels, fmt, n, out, dev)
    return Signal(out, sr, device=str(dev))


def read_wav_batch(paths, device="cuda"):
    """Equal-length, equal-rate files -> ((B, L) float32 CUDA tensor, sample rate)."""
    dev = _require_cuda(device)
    parsed = [_parse_wav(p) for p in paths]
    if not parsed:
        raise ValueError("no files")
    n, sr = parsed[0][4], parsed[0][3]
    if any(p[4] != n or p[3] != sr for p in parsed):
        raise ValueError("read_wav_batch needs files of one length and sample rate")
    out = torch.empty(len(parsed), n, dtype=torch.float32, device=dev)
    for i, (payload, channels, fmt, _, _) in enumerate(parsed):
        _decode_into(payload, channels, fmt, n, out[i], dev)
    return out, sr


def write_spec(path, spec: Spectrogram, dtype: str = "f64") -> None:
    """specfile.py:26-43 -- 32-byte header, then the row-major payload (complex
    cells interleaved re, im) as little-endian float32 or float64."""
    if dtype not in _DTYPE_CODES:
        raise ValueError(f"dtype must be 'f32' or 'f64', got {dtype!r}")
    if spec.kind not in _KIND_CODES:
        raise ValueError(f"unknown spectrogram kind {spec.kind!r}")
    data = spec.data
    if not torch.is_tensor(data):
        data = torch.as_tensor(np.asarray(data))
    if data.is_complex():
        cells = torch.view_as_real(data.to(torch.complex64).contiguous()).reshape(-1)
    else:
        cells = data.to(torch.float32).contiguous().reshape(-1)
    if dtype == "f64" and cells.is_cuda:
        wide = torch.empty(cells.numel(), dtype=torch.float64, device=cells.device)
        L.check(L.load().nnab_widen_f64(cells.data_ptr(), cells.numel(), wide.data_ptr(),
                                        L.stream_handle(cells.device)), "widen_f64")
        blob = wide.cpu().numpy().astype("<f8").tobytes()
    else:
        blob = cells.cpu().numpy().astype("<f8" if dtype == "f64" else "<f4").tobytes()
    header = _HEADER.pack(_MAGIC, _VERSION, _DTYPE_CODES[dtype], _KIND_CODES[spec.kind], 0, int(data.shape[0]),
                          int(data.shape[1]), float(spec.sample_rate), int(spec.hop))
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(blob)


def read_spec(path, device="cuda") -> Spectrogram:
    """specfile.py:46-72 -- the inverse of write_spec (float32 payloads are
    read exactly; float64 payloads are narrowed to the device's float32)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _HEADER.size:
        raise CorruptFileError(f"{path}: shorter than the header")
    magic, version, dtype_code, kind_code, _, n_bins, n_frames, sample_rate, hop = _HEADER.unpack_from(blob, 0)
    if magic != _MAGIC:
        raise CorruptFileError(f"{path}: bad magic {magic!r}")
    if version != _VERSION:
        raise CorruptFileError(f"{path}: unsupported version {version}")
    if kind_code not in _KIND_NAMES or dtype_code not in (0, 1):
        raise CorruptFileError(f"{path}: unknown dtype/kind codes ({dtype_code}, {kind_code})")
    kind = _KIND_NAMES[kind_code]
    scalar = np.dtype("<f4") if dtype_code == 0 else np.dtype("<f8")
    cells = n_bins * n_frames * (2 if kind == "complex" else 1)
    payload = blob[_HEADER.size:]
    if len(payload) != cells * scalar.itemsize:
        raise CorruptFileError(f"{path}: payload is {len(payload)} bytes but the header implies "
                               f"{cells * scalar.itemsize}")
    flat = torch.from_numpy(np.frombuffer(payload, dtype=scalar).astype(np.float32)).to(_require_cuda(device))
    if kind == "complex":
        data = torch.view_as_complex(flat.reshape(n_bins, n_frames, 2).contiguous())
    else:
        data = flat.reshape(n_bins, n_frames)
    return Spectrogram(data=data, bin_freqs_hz=None, hop=hop, sample_rate=sample_rate, kind=kind)
