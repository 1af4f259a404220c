"""Pin the CPU oracle against vectors produced by the real reference.

The oracle (oracle/spectro_oracle.py) is the checker for every GPU parity
test; these CPU tests prove it reproduces `spectro` on the same inputs.
"""

import numpy as np
import pytest

from oracle import spectro_oracle as O

SR = 44100.0
TIGHT = 1e-11  # float64 restatement of float64 reference: rounding-level agreement


def test_pad_kats(golden):
    # tests/test_signal.py:73-79 known answers
    x = np.array([1.0, 2.0, 3.0])
    assert np.array_equal(O.pad(x, 2, 2, "reflect"), golden["pad_reflect_123"])
    assert np.array_equal(O.pad(x, 2, 2, "reflect"), [3, 2, 1, 2, 3, 2, 1])
    assert np.array_equal(O.pad(x, 1, 1, "constant_zero"), golden["pad_zero_123"])
    with pytest.raises(ValueError):
        O.pad(x, 3, 0, "reflect")


def test_pad_index_maps_bit_exact(golden):
    assert np.array_equal(O.pad_index_map(80000, 1024, 1024, "reflect"), golden["padmap_reflect_80000_1024"])
    assert np.array_equal(O.pad_index_map(80000, 11341, 11341, "reflect"), golden["padmap_reflect_80000_11341"])
    assert np.array_equal(O.pad_index_map(100, 7, 7, "constant_zero"), golden["padmap_zero_100_7"])


def test_fir_and_downsample(golden):
    assert np.allclose(O.lowpass_taps(3, 0.5, "rectangular"), golden["fir3_rect"], atol=1e-15)
    assert np.allclose(golden["fir3_rect"], [0.2800496, 0.4399008, 0.2800496], atol=1e-6)
    taps = O.lowpass_taps(255, 0.5, "hamming")
    assert np.array_equal(taps, golden["fir255"])
    got = O.halve_rate(golden["clips"][0].astype(np.float64), taps)
    assert O.peak_err(got, golden["ds2_clip0"]) < TIGHT


def test_banks(golden):
    h_re, h_im = O.stft_bank()
    rows = [0, 1, 17, 512, 1024]
    assert np.array_equal(h_re[rows], golden["dft_h_re_rows"])
    assert np.array_equal(h_im[rows], golden["dft_h_im_rows"])
    assert np.allclose(O.mel_bank(SR, 2048, 128, formula="slaney"), golden["mel_W_slaney"], atol=1e-14)
    assert np.allclose(O.mel_bank(SR, 2048, 128, formula="htk", norm="area"), golden["mel_W_htk_area"],
                       atol=1e-14)
    k, lens = O.cqt_time_bank(O.CqtCfg(sr=SR))
    assert np.array_equal(lens, golden["cqt_lengths"])
    assert k.shape == (84, 22682)  # even(len0), kernels.py:384-388
    assert np.allclose(k[[0, 11, 40, 83]], golden["cqt_rows"], atol=1e-16)
    plan = O.cqt2010_plan(O.CqtCfg(sr=SR))
    assert [plan.n_octaves, plan.early_stages, plan.kernel_hop, plan.first_bin] == list(golden["cqt2010_meta"])
    assert np.allclose(plan.top_kernels, golden["cqt2010_top_kernels"], atol=1e-16)


def test_full_size_configs(golden):
    clips = golden["clips"].astype(np.float64)
    h_re, h_im = O.stft_bank()
    W = O.mel_bank(SR, 2048, 128, formula="slaney")
    kern, _ = O.cqt_time_bank(O.CqtCfg(sr=SR))
    plan = O.cqt2010_plan(O.CqtCfg(sr=SR))
    for i, c in enumerate(clips):
        s = O.stft_clip(c, h_re, h_im, 512)
        assert s.shape == (1025, 157)
        assert O.peak_err(s, golden["stft_mag_full"][i]) < 1e-7  # golden stored as float32
        assert O.peak_err(O.mel_clip(c, h_re, h_im, W, 512), golden["mel_full"][i]) < TIGHT
        assert O.peak_err(O.mel_clip(c, h_re, h_im, W, 512, power=2.0), golden["mel_full_p2"][i]) < TIGHT
        assert O.peak_err(O.cqt1992v2_clip(c, kern, 512), golden["cqt1992v2_full"][i]) < TIGHT
        assert O.peak_err(O.cqt2010v2_clip(c, O.CqtCfg(sr=SR), plan), golden["cqt2010v2_full"][i]) < TIGHT


def test_small_configs(golden):
    xs = golden["small_x"]
    def bank(n_fft, sr, **kw):
        return O.stft_bank(n_fft, sr, **kw)
    h = bank(128, 8000.0)
    assert O.peak_err(O.stft_clip(xs, *h, 64, output="complex"), golden["stft_small_complex"]) < TIGHT
    assert O.peak_err(O.stft_clip(xs, *h, 32, pad_mode="constant_zero", output="power"),
                      golden["stft_small_power_zero"]) < TIGHT
    hh = bank(128, 8000.0, window_kind="hamming")
    assert O.peak_err(O.stft_clip(xs, *hh, 48, center=False), golden["stft_small_nocenter"]) < TIGHT
    hl = bank(256, 8000.0, freq_scale="log", fmin=80.0, fmax=3500.0, freq_bins=100)
    assert O.peak_err(O.stft_clip(xs, *hl, 64), golden["stft_small_log"]) < TIGHT
    hn = bank(256, 8000.0, freq_scale="linear", fmin=50.0, fmax=3000.0, freq_bins=90)
    assert O.peak_err(O.stft_clip(xs, *hn, 64), golden["stft_small_linear"]) < TIGHT
    h2 = bank(256, 8000.0)
    W = O.mel_bank(8000.0, 256, 12, formula="htk")
    assert O.peak_err(O.mel_clip(xs, *h2, W, 128), golden["mel_small_htk"]) < TIGHT
    x22 = golden["x22"]
    k, _ = O.cqt_time_bank(O.CqtCfg(sr=22050.0, fmin=220.0, n_bins=24))
    assert O.peak_err(O.cqt1992v2_clip(x22, k, 512, output="complex"), golden["cqt1992v2_small_complex"]) < TIGHT
    for key, cfg in [("cqt2010v2_small", O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256)),
                     ("cqt2010v2_ragged", O.CqtCfg(sr=22050.0, fmin=82.0, n_bins=50, hop_length=256)),
                     ("cqt2010v2_noearly", O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256,
                                                    early_downsample=False))]:
        assert O.peak_err(O.cqt2010v2_clip(x22, cfg), golden[key]) < TIGHT, key


def test_hop_divisibility():
    # tests/test_transforms.py:283-287
    with pytest.raises(ValueError, match="divisible"):
        O.cqt2010_plan(O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=100))


def test_trainable_vjp(golden):
    xg = golden["grad_x"]
    h_re, h_im = O.stft_bank(32, 8000.0)
    _, _, _, S = O.smooth_mag_forward(xg, h_re, h_im, 32)
    assert O.peak_err(S, golden["grad_stft_S"]) < TIGHT
    g, gx = O.conv_layer_vjp(xg, h_re, h_im, 32, golden["grad_up_stft"], with_input_grad=True)
    assert O.peak_err(g["h_re"], golden["grad_stft_h_re"]) < TIGHT
    assert O.peak_err(g["h_im"], golden["grad_stft_h_im"]) < TIGHT
    assert O.peak_err(gx, golden["grad_stft_x"]) < TIGHT
    h_re, h_im = O.stft_bank(64, 8000.0)
    g, gx = O.conv_layer_vjp(xg, h_re, h_im, 16, golden["grad_up_stft_hop16"], with_input_grad=True)
    assert O.peak_err(g["h_re"], golden["grad_stft_hop16_h_re"]) < TIGHT
    assert O.peak_err(gx, golden["grad_stft_hop16_x"]) < TIGHT
    h_re, h_im = O.stft_bank(32, 8000.0)
    W = O.mel_bank(8000.0, 32, 4, formula="htk")
    assert O.peak_err(O.mel_layer_forward(xg, W, h_re, h_im, 32), golden["grad_mel_fwd"]) < TIGHT
    gm = O.mel_layer_vjp(xg, W, h_re, h_im, 32, golden["grad_up_mel"])
    assert O.peak_err(gm["weights"], golden["grad_mel_W"]) < TIGHT
    k, _ = O.cqt_time_bank(O.CqtCfg(sr=8000.0, fmin=200.0, n_bins=12, hop_length=128))
    gc = O.conv_layer_vjp(golden["grad_xc"], k.real, k.imag, 128, golden["grad_up_cqt"])
    assert O.peak_err(gc["h_re"], golden["grad_cqt_h_re"]) < TIGHT
    assert O.peak_err(gc["h_im"], golden["grad_cqt_h_im"]) < TIGHT


def test_oracle_frequency_domain_cqt_matches_golden(golden):
    """Cqt1992 / Cqt2010 (transforms.py:211-238, 326-337) restated through np.fft."""
    x22 = golden["x22"]
    cfg_s = O.CqtCfg(sr=22050.0, fmin=220.0, n_bins=24, hop_length=512)
    assert O.peak_err(O.cqt1992_clip(x22, cfg_s), golden["cqt1992_small"]) < 1e-10
    assert O.peak_err(O.cqt1992_clip(x22, cfg_s, output="complex"), golden["cqt1992_small_complex"]) < 1e-10
    cfg_r = O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256)
    assert O.peak_err(O.cqt2010_clip(x22, cfg_r), golden["cqt2010_small"]) < 1e-10
    # the reference's documented equivalence with the time-domain variants
    assert O.peak_err(golden["cqt1992_small_complex"], golden["cqt1992v2_small_complex"]) < 1e-9
