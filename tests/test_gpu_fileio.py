"""File formats either side of the hot path:
device-side WAV ingestion against the reference's read_wav (wavio.py:19-68) and
SpecFile output byte-identical to the reference's write_spec (specfile.py:26-43),
on fixtures the reference produced (tests/golden/make_golden.py)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

WAVS = ["wav_pcm16_mono", "wav_float32_mono", "wav_pcm16_stereo", "wav_pcm16_3ch", "wav_f32_stereo"]


@pytest.mark.parametrize("name", WAVS)
def test_read_wav_matches_reference(golden, cuda_dev, tmp_path, name):
    from paper_1912_12055_b200 import fileio
    p = tmp_path / (name + ".wav")
    p.write_bytes(golden[name + "_bytes"].tobytes())
    sig = fileio.read_wav(str(p), device=cuda_dev)
    want = golden[name + "_decoded"]
    got = sig.samples.cpu().numpy()
    assert sig.sample_rate == float(golden[name + "_sr"])
    assert got.shape == want.shape
    if name == "wav_pcm16_3ch":  # /3: the reference rounds to float64 first (double rounding, <= 1 ulp)
        assert np.max(np.abs(got.astype(np.float64) - want) / np.maximum(np.abs(want), 1e-30)) <= 2 ** -23
    else:  # bit-exact to float32(reference)
        assert np.array_equal(got, want.astype(np.float32))


def test_read_wav_batch(golden, cuda_dev, tmp_path):
    from paper_1912_12055_b200 import fileio
    paths = []
    for i in range(3):
        p = tmp_path / f"c{i}.wav"
        p.write_bytes(golden["wav_pcm16_stereo_bytes"].tobytes())
        paths.append(str(p))
    x, sr = fileio.read_wav_batch(paths, device=cuda_dev)
    assert x.shape == (3, golden["wav_pcm16_stereo_decoded"].size) and sr == 16000.0
    assert torch.equal(x[0], x[2])


@pytest.mark.parametrize("name", ["specfile_complex", "specfile_mag"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_write_spec_byte_identical(golden, cuda_dev, tmp_path, name, dtype):
    from paper_1912_12055_b200 import fileio
    from paper_1912_12055_b200.spectro import Spectrogram
    src = golden["stft_small_complex"]
    if name == "specfile_complex":
        data = torch.from_numpy(src.astype(np.complex64)).to(cuda_dev)
        kind = "complex"
    else:
        data = torch.from_numpy(np.abs(src).astype(np.float32)).to(cuda_dev)
        kind = "magnitude"
    spec = Spectrogram(data=data, bin_freqs_hz=None, hop=64, sample_rate=8000.0, kind=kind)
    p = tmp_path / "s.nasp"
    fileio.write_spec(str(p), spec, dtype=dtype)
    assert p.read_bytes() == golden[name + "_" + dtype].tobytes()
    back = fileio.read_spec(str(p), device=cuda_dev)
    assert back.kind == kind and back.hop == 64 and back.sample_rate == 8000.0
    assert torch.equal(back.data, data)


# ---- ports of the reference's SpecFile / WAV tests (tests/test_specfile.py, tests/test_wavio.py)

def _spec(kind="magnitude", n_bins=3, n_frames=4, seed=0, device="cuda:0"):
    from paper_1912_12055_b200.spectro import Spectrogram
    rng = np.random.default_rng(seed)
    if kind == "complex":
        d = (rng.standard_normal((n_bins, n_frames)) + 1j * rng.standard_normal((n_bins, n_frames))).astype(np.complex64)
    else:
        d = np.abs(rng.standard_normal((n_bins, n_frames))).astype(np.float32)
    return Spectrogram(data=torch.from_numpy(d).to(device), bin_freqs_hz=None, hop=512, sample_rate=22050.0, kind=kind)


@pytest.mark.parametrize("kind", ["magnitude", "power", "complex"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_spec_round_trip_exact(cuda_dev, tmp_path, kind, dtype):  # test_specfile.py:21-37
    from paper_1912_12055_b200 import fileio
    spec = _spec(kind)
    p = tmp_path / "s.spec"
    fileio.write_spec(str(p), spec, dtype=dtype)
    back = fileio.read_spec(str(p), device=cuda_dev)
    assert torch.equal(back.data, spec.data)  # float32 cells survive either payload width
    assert back.kind == kind and back.hop == 512 and back.sample_rate == 22050.0


def test_spec_writes_deterministic_and_layout(cuda_dev, tmp_path):  # test_specfile.py:39-69
    import struct
    from paper_1912_12055_b200 import fileio
    spec = _spec("complex")
    a, b = tmp_path / "a.spec", tmp_path / "b.spec"
    fileio.write_spec(str(a), spec)
    fileio.write_spec(str(b), spec)
    assert a.read_bytes() == b.read_bytes()
    p = tmp_path / "p.spec"
    fileio.write_spec(str(p), _spec("power", n_bins=2, n_frames=5))
    blob = p.read_bytes()
    magic, version, dtype, kind, reserved, n_bins, n_frames, sr, hop = struct.unpack_from("<4sIBBHIIdI", blob, 0)
    assert (magic, version, dtype, kind, reserved) == (b"NASP", 1, 1, 1, 0)
    assert (n_bins, n_frames, sr, hop) == (2, 5, 22050.0, 512) and len(blob) == 32 + 2 * 5 * 8
    c = _spec("complex", n_bins=1, n_frames=2)
    fileio.write_spec(str(p), c)
    flat = np.frombuffer(p.read_bytes()[32:], dtype="<f8")
    z = c.data.cpu().numpy()
    assert flat[0] == z[0, 0].real and flat[1] == z[0, 0].imag


def test_spec_validation(cuda_dev, tmp_path):  # test_specfile.py:71-103
    from paper_1912_12055_b200 import fileio
    p = tmp_path / "s.spec"
    fileio.write_spec(str(p), _spec())
    good = p.read_bytes()
    for blob in (b"JUNK" + good[4:], good[:-8], b"NASP", good[:4] + bytes([9]) + good[5:]):
        p.write_bytes(blob)
        with pytest.raises(fileio.CorruptFileError):
            fileio.read_spec(str(p), device=cuda_dev)


def _wav(path, fmt, channels, sr, bits, payload, extra_chunk=False):
    import struct
    block = channels * bits // 8
    fmt_chunk = b"fmt " + struct.pack("<I", 16) + struct.pack("<HHIIHH", fmt, channels, sr, sr * block, block, bits)
    body = b"WAVE" + fmt_chunk
    if extra_chunk:
        body += b"LIST" + struct.pack("<I", 4) + b"INFO"
    body += b"data" + struct.pack("<I", len(payload)) + payload
    path.write_bytes(b"RIFF" + struct.pack("<I", len(body)) + body)


def test_wav_pcm16_scaling_stereo_and_chunks(cuda_dev, tmp_path):  # test_wavio.py:25-45
    from paper_1912_12055_b200 import fileio
    p = tmp_path / "a.wav"
    pcm = np.array([0, 16384, -32768, 32767], dtype="<i2")
    _wav(p, 1, 1, 8000, 16, pcm.tobytes(), extra_chunk=True)
    s = fileio.read_wav(str(p), device=cuda_dev)
    assert np.array_equal(s.samples.cpu().numpy(), pcm.astype(np.float32) / 32768.0) and s.sample_rate == 8000.0
    st = np.array([[100, 300], [-200, 200]], dtype="<i2")
    _wav(p, 1, 2, 8000, 16, st.tobytes())
    s = fileio.read_wav(str(p), device=cuda_dev)
    assert np.array_equal(s.samples.cpu().numpy(), (st.astype(np.float64) / 32768.0).mean(axis=1).astype(np.float32))


def test_wav_errors(cuda_dev, tmp_path):  # test_wavio.py:47-80
    from paper_1912_12055_b200 import fileio
    p = tmp_path / "b.wav"
    _wav(p, 6, 1, 8000, 8, b"\x00" * 4)  # A-law
    with pytest.raises(fileio.UnsupportedFormatError):
        fileio.read_wav(str(p), device=cuda_dev)
    _wav(p, 1, 1, 8000, 24, b"\x00" * 6)
    with pytest.raises(fileio.UnsupportedFormatError):
        fileio.read_wav(str(p), device=cuda_dev)
    p.write_bytes(b"NOPE" + b"\x00" * 40)
    with pytest.raises(fileio.CorruptFileError):
        fileio.read_wav(str(p), device=cuda_dev)
