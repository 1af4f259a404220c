"""Generate golden vectors by running the REAL reference (`spectro`) here.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  The fixtures pin `oracle/spectro_oracle.py`
(tests/test_oracle_golden.py) and, through the oracle, the CUDA path.
Inputs are float32-rounded then upcast, exactly as the GPU parity tests feed
both sides (SURVEY.md section 8c "Parity method").
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import spectro as sp  # noqa: E402  (the real reference)
from spectro.gradients import TrainableLayer, spectrogram_vjp  # noqa: E402
from spectro.training import make_mel_layer, make_stft_layer  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    g = {}
    rng = np.random.default_rng(0)
    clips = f32(rng.standard_normal((2, 80000)) * 0.5)  # bench distribution (cli.py:98-99)
    g["clips"] = clips.astype(np.float32)
    sr = 44100.0

    # --- padding / framing index maps (signal.py:138-156, gradients.py:18-25)
    g["pad_reflect_123"] = sp.pad_signal(sp.Signal([1.0, 2.0, 3.0], 1.0), "reflect", 2, 2).samples
    g["pad_zero_123"] = sp.pad_signal(sp.Signal([1.0, 2.0, 3.0], 1.0), "constant_zero", 1, 1).samples
    from spectro.gradients import _pad_index_map
    g["padmap_reflect_80000_1024"] = _pad_index_map(80000, 1024, "reflect").astype(np.int32)
    g["padmap_reflect_80000_11341"] = _pad_index_map(80000, 11341, "reflect").astype(np.int32)
    g["padmap_zero_100_7"] = _pad_index_map(100, 7, "constant_zero").astype(np.int64)

    # --- FIR (signal.py:186-211) and downsample2 (signal.py:232-247)
    g["fir3_rect"] = sp.design_lowpass_fir(3, 0.5, "rectangular").taps
    g["fir255"] = sp.design_lowpass_fir(255, 0.5, "hamming").taps
    g["ds2_clip0"] = sp.downsample2(sp.Signal(clips[0], sr), sp.design_lowpass_fir(255, 0.5)).samples

    # --- banks
    stft_full = sp.Stft(sp.StftParams(), sr)
    g["dft_h_re_rows"] = stft_full.bank.h_re[[0, 1, 17, 512, 1024]]
    g["dft_h_im_rows"] = stft_full.bank.h_im[[0, 1, 17, 512, 1024]]
    mel_full = sp.MelSpec(sp.MelParams(), sr)
    g["mel_W_slaney"] = mel_full.bank.weights
    g["mel_W_htk_area"] = sp.build_mel_filter_bank(sr, 2048, 128, formula="htk", norm="area").weights
    cqt_cfg = sp.CqtConfig(sr=sr)
    c92 = sp.Cqt1992v2(cqt_cfg)
    g["cqt_lengths"] = np.asarray(c92.bank.lengths)
    g["cqt_rows"] = c92.bank.time_kernels[[0, 11, 40, 83]]
    c10 = sp.Cqt2010v2(cqt_cfg)
    g["cqt2010_top_kernels"] = c10.bank.time_kernels
    g["cqt2010_meta"] = np.array([c10.n_octaves, c10.early_stages, c10.kernel_hop, c10._first_bin])

    # --- full-size configs (BASELINE configs 1-4), both clips
    g["stft_mag_full"] = np.stack([stft_full(sp.Signal(c, sr)).data for c in clips]).astype(np.float32)
    g["stft_mag_full_peak"] = np.array([np.max(np.abs(stft_full(sp.Signal(c, sr)).data)) for c in clips])
    g["mel_full"] = np.stack([mel_full(sp.Signal(c, sr)).data for c in clips])
    mel_p2 = sp.MelSpec(sp.MelParams(power=2.0), sr)
    g["mel_full_p2"] = np.stack([mel_p2(sp.Signal(c, sr)).data for c in clips])
    g["cqt1992v2_full"] = np.stack([c92(sp.Signal(c, sr)).data for c in clips])
    g["cqt2010v2_full"] = np.stack([c10(sp.Signal(c, sr)).data for c in clips])

    # --- small configs (reference unit tests' shapes)
    r2 = np.random.default_rng(17)
    xs = f32(r2.standard_normal(1024))
    g["small_x"] = xs
    g["stft_small_complex"] = sp.stft(sp.Signal(xs, 8000.0),
                                      sp.StftParams(n_fft=128, hop_length=64, output="complex")).data
    g["stft_small_power_zero"] = sp.stft(sp.Signal(xs, 8000.0),
                                         sp.StftParams(n_fft=128, hop_length=32, output="power",
                                                       pad_mode="constant_zero")).data
    g["stft_small_nocenter"] = sp.stft(sp.Signal(xs, 8000.0),
                                       sp.StftParams(n_fft=128, hop_length=48, center=False,
                                                     window="hamming")).data
    g["stft_small_log"] = sp.stft(sp.Signal(xs, 8000.0),
                                  sp.StftParams(n_fft=256, hop_length=64, freq_scale="log",
                                                fmin=80.0, fmax=3500.0, freq_bins=100)).data
    g["stft_small_linear"] = sp.stft(sp.Signal(xs, 8000.0),
                                     sp.StftParams(n_fft=256, hop_length=64, freq_scale="linear",
                                                   fmin=50.0, fmax=3000.0, freq_bins=90)).data
    g["mel_small_htk"] = sp.mel_spectrogram(sp.Signal(xs, 8000.0),
                                            sp.MelParams(n_fft=256, n_mels=12, hop_length=128, htk=True)).data
    cfg_s = sp.CqtConfig(sr=22050.0, fmin=220.0, n_bins=24, bins_per_octave=12, hop_length=512)
    x22 = f32(np.random.default_rng(5).standard_normal(22050))
    g["x22"] = x22
    g["cqt1992v2_small_complex"] = sp.cqt1992v2(sp.Signal(x22, 22050.0), cfg_s, output="complex").data
    cfg_r = sp.CqtConfig(sr=22050.0, fmin=55.0, n_bins=48, bins_per_octave=12, hop_length=256)
    g["cqt2010v2_small"] = sp.cqt2010v2(sp.Signal(x22, 22050.0), cfg_r).data
    cfg_rr = sp.CqtConfig(sr=22050.0, fmin=82.0, n_bins=50, bins_per_octave=12, hop_length=256)
    g["cqt2010v2_ragged"] = sp.cqt2010v2(sp.Signal(x22, 22050.0), cfg_rr).data
    cfg_ne = sp.CqtConfig(sr=22050.0, fmin=55.0, n_bins=48, bins_per_octave=12, hop_length=256,
                          early_downsample=False)
    g["cqt2010v2_noearly"] = sp.cqt2010v2(sp.Signal(x22, 22050.0), cfg_ne).data
    # frequency-domain variants (transforms.py:211-238, 326-337)
    from spectro.transforms import Cqt1992, Cqt2010
    g["cqt1992_small"] = Cqt1992(cfg_s)(sp.Signal(x22, 22050.0)).data
    g["cqt1992_small_complex"] = Cqt1992(cfg_s)(sp.Signal(x22, 22050.0), output="complex").data
    g["cqt2010_small"] = Cqt2010(cfg_r)(sp.Signal(x22, 22050.0)).data

    # --- file formats either side of the path: WAV bytes the
    # reference reads, and SpecFile bytes it writes
    import struct
    import tempfile
    from spectro.specfile import write_spec
    from spectro.wavio import read_wav, write_wav
    from spectro.transforms import Spectrogram

    def crafted_wav(samples_frames, fmt_tag, bits, sr, extra_chunk=True):
        ch = samples_frames.shape[1]
        if fmt_tag == 1:
            payload = samples_frames.astype("<i2").tobytes()
        else:
            payload = samples_frames.astype("<f4").tobytes()
        block = ch * bits // 8
        fmt = struct.pack("<HHIIHH", fmt_tag, ch, sr, sr * block, block, bits)
        body = b"WAVE" + b"fmt " + struct.pack("<I", len(fmt)) + fmt
        if extra_chunk:  # an odd-sized unknown chunk the reader must skip (word alignment)
            body += b"LIST" + struct.pack("<I", 5) + b"abcde" + b"\x00"
        body += b"data" + struct.pack("<I", len(payload)) + payload + (b"\x00" if len(payload) % 2 else b"")
        return b"RIFF" + struct.pack("<I", len(body)) + body

    rw = np.random.default_rng(8)
    wavs = {
        "wav_pcm16_stereo": crafted_wav(rw.integers(-32768, 32768, size=(3001, 2)), 1, 16, 16000),
        "wav_pcm16_3ch": crafted_wav(rw.integers(-32768, 32768, size=(2000, 3)), 1, 16, 22050),
        "wav_f32_stereo": crafted_wav(rw.standard_normal((2500, 2)).astype(np.float32) * 0.3, 3, 32, 44100),
    }
    with tempfile.TemporaryDirectory() as td:
        for enc in ("pcm16", "float32"):
            pth = os.path.join(td, enc + ".wav")
            write_wav(pth, sp.Signal(f32(rw.standard_normal(1999) * 0.2), 8000.0), encoding=enc)
            wavs["wav_" + enc + "_mono"] = open(pth, "rb").read()
        for name, blob in wavs.items():
            pth = os.path.join(td, name + ".wav")
            open(pth, "wb").write(blob)
            sig = read_wav(pth)
            g[name + "_bytes"] = np.frombuffer(blob, dtype=np.uint8).copy()
            g[name + "_decoded"] = np.asarray(sig.samples)
            g[name + "_sr"] = np.array(sig.sample_rate)
        spec_c = Spectrogram(data=g["stft_small_complex"].astype(np.complex64).astype(np.complex128),
                             bin_freqs_hz=None, hop=64, sample_rate=8000.0, kind="complex")
        spec_m = Spectrogram(data=np.abs(g["stft_small_complex"]).astype(np.float32).astype(np.float64),
                             bin_freqs_hz=None, hop=64, sample_rate=8000.0, kind="magnitude")
        for name, spec in (("specfile_complex", spec_c), ("specfile_mag", spec_m)):
            for dt in ("f32", "f64"):
                pth = os.path.join(td, name + dt + ".nasp")
                write_spec(pth, spec, dtype=dt)
                g[name + "_" + dt] = np.frombuffer(open(pth, "rb").read(), dtype=np.uint8).copy()

    # --- trainable layers (gradients.py:28-149)
    xg = f32(np.random.default_rng(4).standard_normal(512))
    g["grad_x"] = xg
    layer = make_stft_layer(8000.0, n_fft=32)
    up = np.random.default_rng(12).standard_normal(layer.spectrogram(sp.Signal(xg, 8000.0)).shape)
    g["grad_up_stft"] = up
    g["grad_stft_S"] = layer.spectrogram(sp.Signal(xg, 8000.0))
    gr, gx = spectrogram_vjp(sp.Signal(xg, 8000.0), layer, up, with_input_grad=True)
    g["grad_stft_h_re"], g["grad_stft_h_im"], g["grad_stft_x"] = gr["h_re"], gr["h_im"], gx
    layer_h = make_stft_layer(8000.0, n_fft=64, hop=16)
    up_h = np.random.default_rng(13).standard_normal(layer_h.spectrogram(sp.Signal(xg, 8000.0)).shape)
    g["grad_up_stft_hop16"] = up_h
    gr, gx = spectrogram_vjp(sp.Signal(xg, 8000.0), layer_h, up_h, with_input_grad=True)
    g["grad_stft_hop16_h_re"], g["grad_stft_hop16_h_im"], g["grad_stft_hop16_x"] = gr["h_re"], gr["h_im"], gx
    mlayer = make_mel_layer(8000.0, n_fft=32, n_mels=4)
    upm = np.random.default_rng(14).standard_normal(mlayer.spectrogram(sp.Signal(xg, 8000.0)).shape)
    g["grad_up_mel"] = upm
    g["grad_mel_fwd"] = mlayer.spectrogram(sp.Signal(xg, 8000.0))
    g["grad_mel_W"] = spectrogram_vjp(sp.Signal(xg, 8000.0), mlayer, upm)["weights"]
    cfg_g = sp.CqtConfig(sr=8000.0, fmin=200.0, n_bins=12, bins_per_octave=12, hop_length=128)
    clayer = TrainableLayer(sp.build_cqt_kernels(cfg_g, domain="time"), hop=128)
    xgc = f32(np.random.default_rng(6).standard_normal(1024))
    g["grad_xc"] = xgc
    upc = np.random.default_rng(15).standard_normal(clayer.spectrogram(sp.Signal(xgc, 8000.0)).shape)
    g["grad_up_cqt"] = upc
    gr = spectrogram_vjp(sp.Signal(xgc, 8000.0), clayer, upc)
    g["grad_cqt_h_re"], g["grad_cqt_h_im"] = gr["h_re"], gr["h_im"]

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
