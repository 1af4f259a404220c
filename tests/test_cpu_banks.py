"""Host-side kernel-bank builders (paper_1912_12055_b200.banks, init-time)
against the reference's own known-answer tests (tests/test_kernels.py)."""

import math

import numpy as np
import pytest

from paper_1912_12055_b200 import banks as K


class TestFrequencyScale:  # tests/test_kernels.py:11-49
    def test_linear_scale_anchor_values(self):
        nf, _ = K.frequency_scale("linear", 2048, 44100.0, 50.0, 6000.0, 1025)
        assert abs(nf[0] - 2.3220) < 5e-5
        assert abs(nf[1] - 2.5916) < 5e-5
        assert abs(nf[1024] - 278.3698777722471) < 1e-9

    def test_integer_scale(self):
        nf, _ = K.frequency_scale("no", 8, 8000.0, 50.0, 6000.0, 5)
        assert np.array_equal(nf, [0, 1, 2, 3, 4])

    def test_log_scale_endpoints(self):
        n, sr, fmin, fmax, bins = 2048, 44100.0, 50.0, 6000.0, 1025
        nf, _ = K.frequency_scale("log", n, sr, fmin, fmax, bins)
        assert abs(nf[0] - fmin * n / sr) < 1e-12
        assert abs(nf[-1] * (nf[1] / nf[0]) - fmax * n / sr) < 1e-9

    def test_linear_and_log_share_endpoints(self):
        n, sr, fmin, fmax, bins = 1024, 16000.0, 100.0, 7000.0, 300
        lin, _ = K.frequency_scale("linear", n, sr, fmin, fmax, bins)
        log, _ = K.frequency_scale("log", n, sr, fmin, fmax, bins)
        assert abs(lin[0] - log[0]) < 1e-12
        assert abs((lin[-1] + (lin[1] - lin[0])) - log[-1] * (log[1] / log[0])) < 1e-9

    def test_errors(self):
        with pytest.raises(ValueError):
            K.frequency_scale("linear", 2048, 44100.0, 6000.0, 50.0, 1025)
        with pytest.raises(ValueError):
            K.frequency_scale("linear", 2048, 44100.0, 50.0, 23000.0, 1025)
        with pytest.raises(ValueError):
            K.frequency_scale("no", 16, 8000.0, 50.0, 6000.0, 10)

    def test_bin_freqs(self):
        _, hz = K.frequency_scale("no", 2048, 44100.0, 50.0, 6000.0, None)
        assert abs(hz[1] - 21.533203125) < 1e-12
        assert hz[1024] == 22050.0


class TestDftKernels:  # tests/test_kernels.py:67-105
    def test_dc_row_rectangular(self):
        h_re, h_im = K.dft_kernels(np.arange(5.0), K.make_window("rectangular", 8))
        assert np.array_equal(h_re[0], np.ones(8)) and not h_im[0].any()

    def test_k1_row(self):
        h_re, h_im = K.dft_kernels(np.arange(5.0), K.make_window("rectangular", 8))
        n = np.arange(8)
        assert np.allclose(h_re[1], np.cos(2 * np.pi * n / 8), atol=1e-15)
        assert np.allclose(h_im[1], np.sin(2 * np.pi * n / 8), atol=1e-15)


class TestMelScale:  # tests/test_kernels.py:108-126
    def test_htk_700(self):
        assert abs(K.hz_to_mel(700.0) - 2595.0 * np.log10(2.0)) < 1e-12

    def test_slaney_breakpoint(self):
        assert abs(K.hz_to_mel(1000.0, "slaney") - 15.0) < 1e-12

    def test_slaney_linear_region(self):
        assert abs(K.hz_to_mel(200.0, "slaney") - 3.0) < 1e-12

    @pytest.mark.parametrize("formula", ["htk", "slaney"])
    @pytest.mark.parametrize("f", [20.0, 440.0, 4186.0, 15000.0])
    def test_round_trip(self, formula, f):
        assert abs(float(K.mel_to_hz(K.hz_to_mel(f, formula), formula)) - f) <= 1e-9 * f

    def test_negative_rejected(self):
        with pytest.raises(ValueError):
            K.hz_to_mel(-1.0)


class TestMelFilterBank:  # tests/test_kernels.py:129-179
    def test_table_mapping(self):
        w, _ = K.mel_filter_bank(1000.0, 128, 4, 0.0, 500.0, formula="htk")
        spans = []
        for row in w:
            nz = np.nonzero(row)[0]
            spans.append((int(nz[0]), int(nz[-1])))
            assert np.array_equal(nz, np.arange(nz[0], nz[-1] + 1))
        assert spans == [(1, 21), (11, 34), (22, 48), (35, 64)]

    def test_peak_one_and_nonnegative(self):
        w, _ = K.mel_filter_bank(16000.0, 512, 20, 0.0, 8000.0, formula="slaney")
        assert (w >= 0.0).all() and np.allclose(w.max(axis=1), 1.0)

    def test_rows_unimodal(self):
        w, _ = K.mel_filter_bank(22050.0, 1024, 24, 30.0, 11025.0, formula="htk")
        for row in w:
            peak = np.argmax(row)
            d = np.diff(row)
            assert (d[:peak] >= -1e-15).all() and (d[peak:] <= 1e-15).all()

    def test_area_norm(self):
        sr, n_fft, n_mels = 16000.0, 2048, 10
        peak, _ = K.mel_filter_bank(sr, n_fft, n_mels, 100.0, 8000.0, "htk", norm="none")
        area, _ = K.mel_filter_bank(sr, n_fft, n_mels, 100.0, 8000.0, "htk", norm="area")
        df = sr / n_fft
        for m in range(n_mels):
            assert abs(area[m].sum() * df - 1.0) < 0.05
            support = area[m] > 0
            ratios = area[m][support] / peak[m][support]
            assert np.max(np.abs(ratios - ratios[0])) < 1e-12 * ratios[0]

    def test_empty_filter_warns(self):
        with pytest.warns(UserWarning):
            K.mel_filter_bank(44100.0, 64, 16, 0.0, 22050.0, formula="htk")

    def test_errors(self):
        with pytest.raises(ValueError):
            K.mel_filter_bank(1000.0, 128, 4, 0.0, 600.0)
        with pytest.raises(ValueError):
            K.mel_filter_bank(1000.0, 128, 0, 0.0, 500.0)


class TestCqtKernels:  # tests/test_kernels.py:182-254
    def test_q_values(self):
        assert abs(K.cqt_q(12) - 16.817153745105756) < 1e-12
        assert abs(K.cqt_q(24) - 34.12708770892056) < 1e-12
        assert K.cqt_q(1) == 1.0
        with pytest.raises(ValueError):
            K.cqt_q(0)

    @staticmethod
    def freqs(fmin, n_bins, bpo):
        return fmin * 2.0 ** (np.arange(n_bins) / bpo)

    def test_piano_range_lengths(self):
        _, lengths = K.cqt_time_kernels(44100.0, self.freqs(27.5, 1, 24), 24, "hann", 1)
        assert int(lengths[0]) in (54727, 54728)

    def test_lengths_strictly_decreasing_and_octave_halving(self):
        _, lengths = K.cqt_time_kernels(22050.0, self.freqs(55.0, 48, 12), 12, "hann", 1)
        assert (np.diff(lengths) < 0).all()
        for k in range(len(lengths) - 12):
            assert abs(int(lengths[k]) - 2 * int(lengths[k + 12])) <= 2

    def test_constant_q_cycle_bound(self):
        f = self.freqs(110.0, 36, 12)
        _, lengths = K.cqt_time_kernels(22050.0, f, 12, "hann", 1)
        cycles = f * lengths / 22050.0
        q = K.cqt_q(12)
        assert (cycles >= q).all() and (cycles < q + f / 22050.0).all()

    def test_norm_variants(self):
        f = self.freqs(220.0, 12, 12)
        l1, _ = K.cqt_time_kernels(8000.0, f, 12, "hann", 1)
        l2, _ = K.cqt_time_kernels(8000.0, f, 12, "hann", 2)
        raw, _ = K.cqt_time_kernels(8000.0, f, 12, "hann", None)
        assert abs(np.abs(l1[0]).sum() - 1.0) < 1e-12
        assert abs(np.sqrt((np.abs(l2[0]) ** 2).sum()) - 1.0) < 1e-12
        assert np.abs(raw[0]).max() <= 1.0 + 1e-12

    def test_kernels_centred_in_even_width(self):
        k, lengths = K.cqt_time_kernels(22050.0, self.freqs(55.0, 48, 12), 12, "hann", 1)
        assert k.shape[1] % 2 == 0
        for r in (0, 20, 47):
            nz = np.nonzero(k[r])[0]
            assert nz[0] == k.shape[1] // 2 - int(lengths[r]) // 2 + 1  # periodic Hann: w[0] = 0

    def test_config_fmax_and_nyquist(self):
        from paper_1912_12055_b200.spectro import CqtConfig
        assert CqtConfig(sr=22050.0, fmin=55.0, n_bins=999, bins_per_octave=12, hop_length=256, fmax=880.0).n_bins == 49
        c = CqtConfig(sr=8000.0, fmin=220.0, n_bins=49, bins_per_octave=12, hop_length=256)
        assert abs(c.bin_freqs_hz[0] - 220.0) < 1e-9 and abs(c.bin_freqs_hz[48] - 3520.0) < 1e-9
        with pytest.raises(ValueError):
            CqtConfig(sr=8000.0, fmin=220.0, n_bins=60, bins_per_octave=12, hop_length=256)
