"""GPU parity: CQT1992v2 (tcgen05 long-bank GEMM) and CQT2010v2 (device octave
recursion) vs the reference's golden vectors and the oracle."""

import numpy as np
import pytest
import torch

from oracle import spectro_oracle as O

pytestmark = pytest.mark.gpu
SR = 44100.0
TOL = {"tf32": 1e-3, "f16": 1e-3, "fp32": 1e-5, "3xtf32": 1e-5}


def long_engine(cfg, precision, **kw):
    from paper_1912_12055_b200.engine import CqtLongEngine
    k, _ = O.cqt_time_bank(cfg)
    return CqtLongEngine(k, cfg.hop_length, cfg.pad_mode, precision=precision, **kw)


def rec_engine(cfg, precision="fp32"):
    from paper_1912_12055_b200.engine import Cqt2010Engine
    p = O.cqt2010_plan(cfg)
    return Cqt2010Engine(p.taps, p.top_kernels, p.early_stages, p.n_octaves, p.kernel_hop, p.first_bin,
                         cfg.bins_per_octave, cfg.n_bins, cfg.pad_mode, precision=precision)


@pytest.mark.parametrize("precision", ["tf32", "f16", "fp32", "3xtf32"])
def test_cqt1992v2_full_config_golden(golden, cuda_dev, precision):
    eng = long_engine(O.CqtCfg(sr=SR), precision)
    x = torch.from_numpy(golden["clips"]).to(cuda_dev)
    got = eng.forward(x, "magnitude").cpu().numpy()
    assert got.shape == (2, 84, 157)
    for i in range(2):
        err = O.peak_err(got[i], golden["cqt1992v2_full"][i])
        assert err <= TOL[precision], (precision, i, err)


@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_cqt1992v2_small_complex_golden(golden, cuda_dev, precision):
    cfg = O.CqtCfg(sr=22050.0, fmin=220.0, n_bins=24)
    eng = long_engine(cfg, precision)
    got = eng.forward(torch.from_numpy(golden["x22"].astype(np.float32)).to(cuda_dev), "complex")[0].cpu().numpy()
    ref = golden["cqt1992v2_small_complex"]
    assert got.shape == ref.shape
    assert O.peak_err(got, ref) <= TOL[precision]


def test_cqt1992v2_dense_schedule_matches_sparse(golden, cuda_dev):
    cfg = O.CqtCfg(sr=SR)
    a = long_engine(cfg, "fp32")
    b = long_engine(cfg, "fp32", dense=True)
    x = torch.from_numpy(golden["clips"]).to(cuda_dev)
    assert O.peak_err(a.forward(x).cpu().numpy(), b.forward(x).cpu().numpy()) < 1e-5  # accumulation order only


@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_cqt2010v2_full_config_golden(golden, cuda_dev, precision):
    # tf32: fused tensor-core chain (cqt2010_tc.cu); fp32: CUDA-core stage kernels
    eng = rec_engine(O.CqtCfg(sr=SR), precision)
    x = torch.from_numpy(golden["clips"]).to(cuda_dev)
    got = eng.forward(x, "magnitude").cpu().numpy()
    assert got.shape == (2, 84, 157)
    for i in range(2):
        err = O.peak_err(got[i], golden["cqt2010v2_full"][i])
        assert err <= TOL[precision], (precision, i, err)


@pytest.mark.parametrize("key,cfg", [
    ("cqt2010v2_small", O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256)),
    ("cqt2010v2_ragged", O.CqtCfg(sr=22050.0, fmin=82.0, n_bins=50, hop_length=256)),
    ("cqt2010v2_noearly", O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256, early_downsample=False)),
])
@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_cqt2010v2_small_golden(golden, cuda_dev, key, cfg, precision):
    eng = rec_engine(cfg, precision)
    got = eng.forward(torch.from_numpy(golden["x22"].astype(np.float32)).to(cuda_dev))[0].cpu().numpy()
    ref = golden[key]
    assert got.shape == ref.shape
    assert O.peak_err(got, ref) <= TOL[precision]


@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_cqt2010v2_batch_matches_oracle(cuda_dev, precision):
    cfg = O.CqtCfg(sr=SR)
    rng = np.random.default_rng(9)
    x = (rng.standard_normal((5, 80000)) * 0.5).astype(np.float32)
    plan = O.cqt2010_plan(cfg)
    ref = O.map_clips(lambda c: O.cqt2010v2_clip(c.astype(np.float64), cfg, plan), x, threads=4)
    got = rec_engine(cfg, precision).forward(torch.from_numpy(x).to(cuda_dev)).cpu().numpy()
    for i in range(5):  # peak-normalised per clip, as the reference tests do
        assert O.peak_err(got[i], ref[i]) <= TOL[precision], (i, O.peak_err(got[i], ref[i]))
    z = rec_engine(cfg, precision).forward(torch.zeros(2, 80000, device=cuda_dev))
    assert not z.any()
    # odd length and a sweep tone through the same fused path
    t = np.arange(80001) / SR
    sweep = np.sin(2 * np.pi * (40.0 * t + 2000.0 * t * t)).astype(np.float32)
    ref2 = O.cqt2010v2_clip(sweep.astype(np.float64), cfg, plan)
    got2 = rec_engine(cfg, precision).forward(torch.from_numpy(sweep).to(cuda_dev))[0].cpu().numpy()
    assert O.peak_err(got2, ref2) <= TOL[precision]


def test_cqt_host_paths_match_device(cuda_dev):
    """The C-ABI host entry points (pinned buffers, chunked H2D / compute / D2H)
    give the device path's results, including a ragged last chunk."""
    cfg = O.CqtCfg(sr=SR)
    rng = np.random.default_rng(3)
    x = torch.from_numpy((rng.standard_normal((7, 80000)) * 0.5).astype(np.float32))
    xh = x.pin_memory()
    e1 = long_engine(cfg, "tf32")
    want = e1.forward(x.to(cuda_dev)).cpu()
    got = e1.forward_host(xh, chunk_clips=3)
    torch.cuda.synchronize()
    # the hybrid's E-GEMM sums each output's hop-offset terms in an order set by
    # the slot's position in its 128-slot tile, which moves with the chunking
    assert O.peak_err(got.numpy(), want.numpy()) < 1e-6
    e1s = long_engine(cfg, "tf32", method="schedule")
    want_s = e1s.forward(x.to(cuda_dev)).cpu()
    got_s = e1s.forward_host(xh, chunk_clips=3)
    torch.cuda.synchronize()
    assert torch.equal(got_s, want_s)
    e2 = rec_engine(cfg, "tf32")
    want2 = e2.forward(x.to(cuda_dev)).cpu()
    got2 = e2.forward_host(xh, chunk_clips=3)
    torch.cuda.synchronize()
    assert torch.equal(got2, want2)


@pytest.mark.parametrize("case", ["quiet", "loud", "impulse", "silence_spike", "tone"])
def test_cqt2010v2_fp16_scaling_robust(cuda_dev, case):
    """The fused chain runs FP16 operands under an exact per-clip power-of-two
    scale: clips far from unit amplitude, sparse spikes and constant signals stay
    within the TF32-mode tolerance (peak-normalised, like the reference tests)."""
    cfg = O.CqtCfg(sr=SR)
    rng = np.random.default_rng(11)
    n = 80000
    if case == "quiet":
        x = rng.standard_normal(n) * 1e-6
    elif case == "loud":
        x = rng.standard_normal(n) * 2e4
    elif case == "impulse":
        x = np.zeros(n)
        x[40000] = 1.0
    elif case == "silence_spike":
        x = rng.standard_normal(n) * 1e-8
        x[61234] = 3.0
    else:  # (a constant input is not a case: its CQT is ~3e-5 of the input, below any 11-bit-operand mode)
        x = 0.8 * np.sin(2 * np.pi * 440.0 * np.arange(n) / SR)
    x = x.astype(np.float32)
    ref = O.cqt2010v2_clip(x.astype(np.float64), cfg, O.cqt2010_plan(cfg))
    got = rec_engine(cfg, "tf32").forward(torch.from_numpy(x).to(cuda_dev))[0].cpu().numpy()
    assert np.isfinite(got).all()
    assert O.peak_err(got, ref) <= TOL["tf32"], O.peak_err(got, ref)


@pytest.mark.parametrize("method", ["egemm", "hybrid"])
def test_cqt1992v2_egemm_matches_schedule(golden, cuda_dev, method):
    """The hop-offset GEMM (csrc/cqt1992_egemm.cu), alone or for the long bins
    of the hybrid, and the per-K-block schedule (csrc/cqt1992.cu) compute the
    same TF32 correlation in different orders."""
    cfg = O.CqtCfg(sr=SR)
    x = torch.from_numpy(golden["clips"]).to(cuda_dev)
    a = long_engine(cfg, "tf32", method=method)
    if method == "egemm":
        assert a.egemm is not None
    else:
        assert a.hybrid is not None and 0 < a.hybrid[-1] < cfg.n_bins
    b = long_engine(cfg, "tf32", method="schedule")
    for kind in ("magnitude", "power", "complex"):
        ga, gb = a.forward(x, kind).cpu().numpy(), b.forward(x, kind).cpu().numpy()
        assert O.peak_err(ga, gb) < 5e-4, (kind, O.peak_err(ga, gb))
    # the long bins' E-GEMM output lands in rows [0, n_long), the schedule's after them
    if method == "hybrid":
        n_long = a.hybrid[-1]
        ga, gb = a.forward(x).cpu().numpy(), b.forward(x).cpu().numpy()
        for rows in (slice(0, n_long), slice(n_long, cfg.n_bins)):
            assert O.peak_err(ga[:, rows], gb[:, rows]) < 5e-4


def test_cqt1992v2_default_is_hybrid(cuda_dev):
    cfg = O.CqtCfg(sr=SR)
    e = long_engine(cfg, "tf32")
    assert e.hybrid is not None
    assert long_engine(cfg, "3xtf32").hybrid is not None  # FP32-accurate mode: 3xTF32 E-GEMM + schedule


def test_cqt1992v2_hybrid_3xtf32_matches_oracle(golden, cuda_dev):
    """The 3xTF32 hybrid (E-GEMM with main + correction accumulators) at the FP32
    tolerance, against the schedule in the same precision and the golden output."""
    cfg = O.CqtCfg(sr=SR)
    x = torch.from_numpy(golden["clips"]).to(cuda_dev)
    a = long_engine(cfg, "3xtf32")
    b = long_engine(cfg, "3xtf32", method="schedule")
    for kind in ("magnitude", "complex"):
        ga, gb = a.forward(x, kind).cpu().numpy(), b.forward(x, kind).cpu().numpy()
        assert O.peak_err(ga, gb) < 1e-5, (kind, O.peak_err(ga, gb))
    assert O.peak_err(a.forward(x).cpu().numpy(), golden["cqt1992v2_full"]) <= 1e-5


def test_frequency_domain_variants_golden(golden, cuda_dev):
    """spectro.Cqt1992 / Cqt2010 (the reference's frequency-domain routes,
    transforms.py:211-238 and 326-337) against the reference's own outputs."""
    from paper_1912_12055_b200 import spectro as S
    x = S.Signal(golden["x22"].astype(np.float32), 22050.0, device="cuda:0")
    c1 = S.Cqt1992(S.CqtConfig(sr=22050.0, fmin=220.0, n_bins=24, hop_length=512))
    assert O.peak_err(c1(x).data.cpu().numpy(), golden["cqt1992_small"]) <= TOL["tf32"]
    assert O.peak_err(c1(x, "complex").data.cpu().numpy(), golden["cqt1992_small_complex"]) <= TOL["tf32"]
    c2 = S.Cqt2010(S.CqtConfig(sr=22050.0, fmin=55.0, n_bins=48, hop_length=256))
    assert O.peak_err(c2(x).data.cpu().numpy(), golden["cqt2010_small"]) <= TOL["tf32"]
    # the frequency route's fft_len // 2 reflect pad rejects signals the v2 route accepts
    short = S.Signal(golden["x22"][:1000].astype(np.float32), 22050.0, device="cuda:0")  # fft_len 2048 > 2 * 1000 > width 1686
    with pytest.raises(ValueError):
        c1(short)


@pytest.mark.parametrize("fmin,n_bins,bpo,length,batch", [
    (32.70, 84, 12, 30000, 3),     # short clips: fewer hop rows than an M tile per clip
    (55.0, 60, 12, 80001, 2),      # odd length, shorter bank
    (27.5, 96, 24, 50000, 1),      # 24 bins per octave: many long bins, one clip
])
def test_cqt1992v2_hybrid_shapes(cuda_dev, fmin, n_bins, bpo, length, batch):
    """Hybrid (E-GEMM long bins + schedule short bins) against the schedule on
    other banks, ragged lengths and small batches (E-GEMM CTA pairs then walk
    tiles past the data, which must emit nothing)."""
    cfg = O.CqtCfg(sr=SR, fmin=fmin, n_bins=n_bins, bins_per_octave=bpo)
    rng = np.random.default_rng(11)
    x = torch.from_numpy((rng.standard_normal((batch, length)) * 0.5).astype(np.float32)).to(cuda_dev)
    a = long_engine(cfg, "tf32")
    b = long_engine(cfg, "tf32", method="schedule")
    for kind in ("magnitude", "complex"):
        ga, gb = a.forward(x, kind).cpu().numpy(), b.forward(x, kind).cpu().numpy()
        assert np.isfinite(ga).all()
        assert O.peak_err(ga, gb) < 5e-4, (kind, O.peak_err(ga, gb))


def test_cqt1992v2_batch_vs_sequential(golden, cuda_dev):
    """batch == sequential (tests/test_transforms.py:325-342): bit-exact for the
    per-K-block schedule; the hybrid's E-GEMM sums each output's hop-offset terms
    in an order fixed by the slot's absolute position (32-row blocks), so a clip
    moved inside the batch can differ in the last bits (documented in DESIGN.md)."""
    cfg = O.CqtCfg(sr=SR)
    x = torch.from_numpy(golden["clips"]).to(cuda_dev)
    for method in ("schedule", "hybrid"):
        e = long_engine(cfg, "tf32", method=method)
        whole = e.forward(x).cpu().numpy()
        one = np.stack([e.forward(x[i:i + 1])[0].cpu().numpy() for i in range(x.shape[0])])
        if method == "schedule":
            assert np.array_equal(one, whole)
        else:
            assert O.peak_err(one, whole) < 1e-6
        # and run to run, the same launch is bit-reproducible
        assert np.array_equal(e.forward(x).cpu().numpy(), whole)


@pytest.mark.parametrize("mode", ["0", "1", "2", "3-noback"])
def test_cqt2010v2_levels_path_matches_oracle(tmp_path, mode):
    """The CQT2010v2 routes other than the default (front kernel + octave chain + batched
    convs): NNAB_CQT2010_LEVELS=0, the single fused kernel with its convs; =1, the fused
    kernel's front for stages 1-2, level-synchronous HALVE launches and one CONV launch over
    all octaves; =2, the fused kernel through the halvings + the batched convs -- against
    the oracle; 3-noback: the default front with the separate octave-chain and conv launches
    (NNAB_CQT2010_NOBACK=1, the route when the merged back-end kernel is out of reach) -- in a
    subprocess (the switches are read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys; sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from oracle import spectro_oracle as O
from paper_1912_12055_b200.engine import Cqt2010Engine
cfg = O.CqtCfg(sr=44100.0); p = O.cqt2010_plan(cfg)
eng = Cqt2010Engine(p.taps, p.top_kernels, p.early_stages, p.n_octaves, p.kernel_hop, p.first_bin, 12, 84,
                    "reflect", precision="f16")
rng = np.random.default_rng(13)
x = (rng.standard_normal((300, 80000)) * 0.5).astype(np.float32)
x[7] *= 1e-4
got = eng.forward(torch.from_numpy(x).cuda()).cpu().numpy()
errs = [O.peak_err(got[i], O.cqt2010v2_clip(x[i].astype(np.float64), cfg, p)) for i in (0, 7, 150, 299)]
np.save(sys.argv[2], got[:4])
print(max(errs))
'''
    out = str(tmp_path / "lv.npy")
    env = dict(os.environ, NNAB_CQT2010_LEVELS=mode[0])
    if mode == "3-noback":
        env["NNAB_CQT2010_NOBACK"] = "1"
    r = subprocess.run([sys.executable, "-c", code, root, out], env=env, capture_output=True, text=True, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= 1e-3


@pytest.mark.parametrize("precision", ["f16", "fp32"])
def test_cqt1992v2_f16_modes_small_and_ragged(golden, cuda_dev, precision):
    """FP16-operand hybrid (f16, and fp32 = 3xF16): other banks, ragged lengths, a batch
    mixing amplitudes 1e-6 .. 1e4 (per-clip scales) against the oracle."""
    from paper_1912_12055_b200.engine import CqtLongEngine
    for cfg, n in [(O.CqtCfg(sr=22050.0, fmin=55.0, n_bins=48, hop_length=512), 22050),
                   (O.CqtCfg(sr=44100.0, fmin=65.4, n_bins=60, hop_length=512), 50001)]:
        kern, _ = O.cqt_time_bank(cfg)
        eng = CqtLongEngine(kern, 512, "reflect", precision=precision)
        assert eng.hybrid is not None
        rng = np.random.default_rng(21)
        amps = [1e-6, 1.0, 1e4]
        x = np.stack([rng.standard_normal(n) * a for a in amps]).astype(np.float32)
        got = eng.forward(torch.from_numpy(x).to(cuda_dev)).cpu().numpy()
        for i in range(len(amps)):
            ref = O.cqt1992v2_clip(x[i].astype(np.float64), kern, 512)
            assert O.peak_err(got[i], ref) <= TOL[precision], (cfg.n_bins, i, O.peak_err(got[i], ref))


def test_cqt2010v2_mixed_batch_fast_and_exact_scales(cuda_dev):
    """The front kernel's fast scale (from each clip's first 2,048 samples) and its exact
    relaunch for the clips it flags (a silent start, a later peak beyond the headroom), in
    one batch: every clip against the oracle, the silent one exactly zero."""
    cfg = O.CqtCfg(sr=SR)
    plan = O.cqt2010_plan(cfg)
    rng = np.random.default_rng(17)
    n = 80000
    xs = [rng.standard_normal(n) * 0.5,                                           # fast scale
          np.concatenate([np.zeros(5000), rng.standard_normal(n - 5000)]),        # zero start: flagged
          np.concatenate([rng.standard_normal(3000) * 1e-7, rng.standard_normal(n - 3000) * 3.0]),  # flagged
          rng.standard_normal(n) * 1e-6,                                          # fast, quiet
          np.zeros(n),                                                            # all zero: flagged
          rng.standard_normal(n) * 2e4]                                           # fast, loud
    x = np.stack(xs).astype(np.float32)
    got = rec_engine(cfg, "tf32").forward(torch.from_numpy(x).to(cuda_dev)).cpu().numpy()
    assert np.isfinite(got).all()
    assert not got[4].any()
    for i in (0, 1, 2, 3, 5):
        ref = O.cqt2010v2_clip(x[i].astype(np.float64), cfg, plan)
        assert O.peak_err(got[i], ref) <= TOL["tf32"], (i, O.peak_err(got[i], ref))
