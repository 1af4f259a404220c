"""GPU: the reference's signal primitives (signal.py) through the spectro shim,
mirroring the reference's own known-answer tests (tests/test_signal.py) with
the north_star tolerances where the reference asserts float64 ulps."""

import numpy as np
import pytest
import torch

from oracle import spectro_oracle as O

pytestmark = pytest.mark.gpu


def sig(v, sr=1000.0):
    from paper_1912_12055_b200 import spectro as S
    return S.Signal(np.asarray(v, dtype=np.float32), sr, device="cuda:0")


def host(t):
    return t.detach().cpu().numpy()


class TestPadSignal:  # tests/test_signal.py:71-92
    def test_reflect_mirrors_without_edge(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.pad_signal(sig([1.0, 2.0, 3.0]), "reflect", 2, 2)
        assert np.array_equal(host(out.samples), [3, 2, 1, 2, 3, 2, 1])

    def test_zero_pad(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.pad_signal(sig([1.0, 2.0, 3.0]), "constant_zero", 1, 1)
        assert np.array_equal(host(out.samples), [0, 1, 2, 3, 0])

    def test_identity(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        assert np.array_equal(host(S.pad_signal(sig([5.0]), "reflect", 0, 0).samples), [5.0])

    def test_errors(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        with pytest.raises(ValueError):
            S.pad_signal(sig([1.0, 2.0, 3.0]), "reflect", 3, 0)
        with pytest.raises(ValueError):
            S.pad_signal(sig([1.0, 2.0]), "constant_zero", -1, 0)
        with pytest.raises(ValueError):
            S.pad_signal(sig([1.0, 2.0]), "wrap", 1, 1)

    @pytest.mark.parametrize("key,n,pad,mode", [("padmap_reflect_80000_1024", 80000, 1024, "reflect"),
                                                ("padmap_reflect_80000_11341", 80000, 11341, "reflect"),
                                                ("padmap_zero_100_7", 100, 7, "constant_zero")])
    def test_index_map_golden(self, golden, cuda_dev, key, n, pad, mode):
        """The padding index map, bit-exact against np.pad run by the reference
        (gradients.py:18-25 golden): pad arange(n) + 1 (so zero pads stay 0)."""
        from paper_1912_12055_b200 import spectro as S
        out = host(S.pad_signal(sig(np.arange(n) + 1.0), mode, pad, pad).samples).astype(np.int64) - 1
        want = golden[key].astype(np.int64)
        if mode == "constant_zero":
            want = np.where(want < 0, -1, want)
        assert np.array_equal(out, want)


class TestConv1dStrided:  # tests/test_signal.py:95-135
    def test_sliding_sum(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.conv1d_strided(sig([1.0, 2.0, 3.0, 4.0]), [[1.0, 1.0]], 1)
        assert np.allclose(host(out.values), [[3.0, 5.0, 7.0]], rtol=1e-6, atol=0)

    def test_stride_picks_hop_samples(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.conv1d_strided(sig([1.0, 2.0, 3.0, 4.0]), [[1.0, 0.0]], 2)
        assert np.allclose(host(out.values), [[1.0, 3.0]], rtol=1e-6, atol=0)
        assert out.hop == 2

    def test_zero_signal(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.conv1d_strided(sig(np.zeros(16)), [[0.3, -1.0, 2.0], [1.0, 1.0, 1.0]], 3)
        assert not host(out.values).any()

    @pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("tf32", 1e-3)])
    def test_matches_oracle_and_subsampling(self, cuda_dev, precision, tol):
        from paper_1912_12055_b200 import spectro as S
        rng = np.random.default_rng(3)
        x = rng.standard_normal(3000).astype(np.float32)
        kernels = rng.standard_normal((5, 96)).astype(np.float32)
        full = host(S.conv1d_strided(sig(x), kernels, 1, precision=precision).values)
        ref = O.strided_correlate(x.astype(np.float64), kernels.astype(np.float64), 1)
        assert full.shape == ref.shape
        assert O.peak_err(full, ref) <= tol
        for stride in (2, 3, 7, 64):
            hopped = host(S.conv1d_strided(sig(x), kernels, stride, precision=precision).values)
            assert hopped.shape[1] == (3000 - 96) // stride + 1
            assert O.peak_err(hopped, full[:, ::stride][:, :hopped.shape[1]]) <= tol

    def test_linearity(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        rng = np.random.default_rng(11)
        x, y = rng.standard_normal(200), rng.standard_normal(200)
        kernels = rng.standard_normal((4, 16))
        a, b = 1.7, -0.3
        lhs = host(S.conv1d_strided(sig(a * x + b * y), kernels, 8).values)
        rhs = a * host(S.conv1d_strided(sig(x), kernels, 8).values) + b * host(S.conv1d_strided(sig(y), kernels, 8).values)
        assert np.max(np.abs(lhs - rhs)) <= 1e-5 * np.max(np.abs(rhs))

    def test_errors(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        with pytest.raises(ValueError):
            S.conv1d_strided(sig(np.zeros(8)), np.ones((1, 9)), 1)
        with pytest.raises(ValueError):
            S.conv1d_strided(sig(np.zeros(8)), np.ones((1, 4)), 0)
        with pytest.raises(ValueError):
            S.conv1d_strided(sig(np.zeros(8)), np.ones((1, 4)) * 1j, 1)
        with pytest.raises(ValueError):
            S.conv1d_strided(sig(np.zeros(8)), np.zeros((0, 4)), 1)


class TestDownsample2:  # tests/test_signal.py:185-243
    def test_golden_full_clip(self, golden, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.downsample2(sig(golden["clips"][0], 44100.0), S.design_lowpass_fir(255, 0.5))
        assert out.sample_rate == 22050.0
        assert O.peak_err(host(out.samples), golden["ds2_clip0"]) <= 1e-5

    def test_constant_signal_stays_constant(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.downsample2(sig(np.ones(400), 2000.0), S.design_lowpass_fir(31, 0.5, "hamming"))
        assert np.max(np.abs(host(out.samples)[16:-16] - 1.0)) < 1e-6
        assert out.sample_rate == 1000.0 and len(out) == 200

    def test_zero_signal(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        out = S.downsample2(sig(np.zeros(101)), S.design_lowpass_fir(31, 0.5, "hamming"))
        assert not host(out.samples).any() and len(out) == 51

    def test_high_tone_attenuated_50db(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        sr, n = 2000.0, 8192
        x = np.sin(2 * np.pi * (0.9 * sr / 2) * np.arange(n) / sr)
        out = host(S.downsample2(sig(x, sr), S.design_lowpass_fir(255, 0.5, "hamming")).samples)
        assert np.sqrt(np.mean(out[256:-256] ** 2)) < 10 ** (-50 / 20) * np.sqrt(np.mean(x ** 2))

    def test_asymmetric_taps_follow_np_convolve(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        rng = np.random.default_rng(5)
        x = rng.standard_normal(1001)
        taps = rng.standard_normal(9)
        out = host(S.downsample2(sig(x), taps).samples)
        ref = O.halve_rate(x.astype(np.float32).astype(np.float64), taps)
        assert O.peak_err(out, ref) <= 1e-5

    def test_errors(self, cuda_dev):
        from paper_1912_12055_b200 import spectro as S
        with pytest.raises(ValueError):
            S.downsample2(sig(np.zeros(30)), S.design_lowpass_fir(31, 0.5, "hamming"))
        with pytest.raises(ValueError):
            S.downsample2(sig(np.zeros(30)), np.ones(4))
