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
