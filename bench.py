#!/usr/bin/env python
"""Benchmark: spectrograms/s on the 1,770-clip x 80,000-sample batch (44.1 kHz)
plus the roofline fraction of the dominant kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload mel|melpow2|stft|cqt1992v2|cqt2010v2|train]
    python bench.py --impl reference ...     # the reference spectro (baseline/_ref) on the host cores

A step is one pass of the workload over one full batch already resident in
HBM (566 MB of input > 126 MB L2, so no L2 flush is needed between steps).
Multi-GPU: one process per GPU (torchrun); the 1,770 clips are sharded over the
ranks (strong scaling, dist.shard_range; no collective on the forward path,
one bucketed gradient all-reduce in the train workload); `value` = 1,770 clips /
max-over-ranks step time.  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU leg: reference's fastest config

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_CLIPS, L_SAMPLES, SR = 1770, 80000, 44100.0
T_FRAMES = 157
M_FRAMES = B_CLIPS * T_FRAMES  # 277,890

# Algorithmic work per batch; the roofline numerators.
FLOP_STFT = 2.0 * M_FRAMES * 2048 * 2050
FLOP_MEL = FLOP_STFT + 2.0 * M_FRAMES * 1025 * 128
CQT_NONZERO_TAPS = None  # filled from the bank (sum of kernel lengths), 400,975 at the default config
BYTES_CQT2010 = B_CLIPS * L_SAMPLES * 4 + B_CLIPS * 84 * T_FRAMES * 4  # 659.8 MB

WORKLOADS = {
    "stft": "STFT n_fft=2048 hop=512 hann center reflect, magnitude (BASELINE config 1)",
    "mel": "MelSpectrogram n_fft=2048 n_mels=128 hop=512 slaney norm=none power=1, fused (BASELINE config 2)",
    "melpow2": "MelSpectrogram n_fft=2048 n_mels=128 hop=512 slaney norm=none power=2, fused power + mel_basis "
               "epilogue (BASELINE config 2, 'fused power')",
    "cqt1992v2": "CQT1992v2 84 bins 12/oct fmin=32.70 hop=512, magnitude (BASELINE config 3)",
    "cqt2010v2": "CQT2010v2 84 bins 12/oct fmin=32.70 hop=512 early downsample, magnitude (BASELINE config 4)",
    "train": "trainable STFT+Mel (trainable_mel + trainable_STFT, n_fft=2048 n_mels=128 hop=512) forward + "
             "backward (dW, dS, dh) + NCCL kernel-grad all-reduce (BASELINE config 5)",
}
FLOP_TRAIN = FLOP_MEL + 2.0 * M_FRAMES * 2048 * 2050 + 2 * (2.0 * M_FRAMES * 1025 * 128)  # 4.886e12 (section 8d)


class TrainStep:
    """One optimisation step's compute for config 5: forward of the trainable
    Mel layer, backward for the mel weights and both DFT banks, and (N > 1)
    the gradient all-reduce (bucketed, overlapped with the backward GEMMs)."""

    def __init__(self, device, precision, world, nb=B_CLIPS, phasor="split"):
        import torch
        from paper_1912_12055_b200.dist import GradReducer
        from paper_1912_12055_b200.layers import MelSpectrogram
        self.m = MelSpectrogram(sr=SR, n_fft=2048, n_mels=128, hop_length=512, trainable_mel=True,
                                trainable_STFT=True, precision=precision, device=device, grad_phasor=phasor)
        self.world = world
        self.reducer = GradReducer(list(self.m.parameters())) if world > 1 else None
        gen = torch.Generator(device=device)
        gen.manual_seed(77)
        self.g = torch.randn(nb, 128, T_FRAMES, device=device, generator=gen) * 1e-3

    def forward(self, x, kind=None):
        for p in self.m.parameters():
            p.grad = None
        out = self.m(x)
        if self.reducer is not None:
            self.reducer.arm()
        out.backward(self.g)
        if self.reducer is not None:
            self.reducer.finish()
        return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md
    recipe): an NVML thread polling every 2 ms (the timed regions are tens of ms, shorter
    than nvidia-smi's first sample), falling back to `nvidia-smi -lms 25`."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.proc, self.path, self.thread = index, None, f"/tmp/nnab_clocks_{os.getpid()}.csv", None
        self.samples, self.reasons, self.max_mhz = [], set(), 0.0

    def start(self):
        try:
            import threading

            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.stop_flag = False

            def run():
                while not self.stop_flag:
                    self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for n, bit in bits.items():
                        if r & bit:
                            self.reasons.add(n)
                    time.sleep(0.002)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "25"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join(timeout=2)
            if not self.samples:
                return None
            return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML, 2 ms"}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(self.NAMES, parts[2:]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi -lms 25"}


# ------------------------------------------------------------------ workloads
# Operand modes per workload: the engine precision a bench mode maps to, the dtype
# label, and the tensor peak it is measured against ("f16": dense FP16 = measured bf16;
# "tf32": half of it).  "f16" is each transform's fastest <= 1e-3 mode (FP16 operands
# under exact power-of-two scales where the transform has it, else TF32); "fp32" its
# <= 1e-5 mode.
MODES = {
    ("stft", "f16"): ("f16", "f16 operands (exact per-clip / per-bank power-of-two scales), f32 accumulate", "f16"),
    ("stft", "tf32"): ("tf32", "tf32", "tf32"),
    ("stft", "fp32"): ("fp32", "3xf16 (FP16 hi/lo split, exact power-of-two scales, f32 accumulate)", "f16"),
    ("stft", "3xtf32"): ("3xtf32", "3xtf32", "tf32"),
    ("cqt1992v2", "f16"): ("f16", "f16 operands (exact per-clip / per-bank power-of-two scales), f32 accumulate", "f16"),
    ("cqt1992v2", "tf32"): ("tf32", "tf32", "tf32"),
    ("cqt1992v2", "fp32"): ("fp32", "3xf16 (FP16 hi/lo split, exact power-of-two scales, f32 accumulate)", "f16"),
    ("cqt1992v2", "3xtf32"): ("3xtf32", "3xtf32", "tf32"),
    ("cqt2010v2", "f16"): ("f16", "f16 operands (exact per-clip power-of-two scale), f32 accumulate", None),
    ("cqt2010v2", "tf32"): ("f16", "f16 operands (exact per-clip power-of-two scale), f32 accumulate", None),
    ("cqt2010v2", "fp32"): ("fp32", "f32 (CUDA cores)", None),
    # training: the dominant GEMMs (forward, kernel gradient) run on FP16 tensor cores, so the
    # roofline divides by the FP16 (= bf16) peak -- conservative for the TF32 reductions in the step
    ("train", "f16"): ("tf32", "tf32-accurate: 3xf16 forward (phasor), one-pass fp16 kernel gradient (exact "
                               "power-of-two scales), tf32 reductions, f32 accumulate", "f16"),
    ("train", "tf32"): ("tf32", "tf32-accurate: 3xf16 forward (phasor), one-pass fp16 kernel gradient (exact "
                                "power-of-two scales), tf32 reductions, f32 accumulate", "f16"),
    ("train", "fp32"): ("fp32", "fp32-accurate: 3xf16 forward and kernel gradient, 3xtf32 reductions, f32 accumulate",
                        "f16"),
    # TF32 training with the one-pass forward phasor (faster; gradient tail)
    ("train", "tf32-onepass"): ("tf32", "f16 forward (one-pass phasor), one-pass fp16 kernel gradient, tf32 "
                                        "reductions, f32 accumulate", "f16"),
}
for _m in ("f16", "tf32", "fp32", "3xtf32"):
    if ("stft", _m) in MODES:
        MODES[("mel", _m)] = MODES[("melpow2", _m)] = MODES[("stft", _m)]
BREAKDOWN_MODES = {"stft": ["f16", "tf32", "fp32"], "mel": ["f16", "tf32", "fp32"], "melpow2": ["f16", "tf32", "fp32"],
                   "cqt1992v2": ["f16", "tf32", "fp32"], "cqt2010v2": ["f16", "fp32"],
                   "train": ["tf32", "tf32-onepass", "fp32"]}


def build_workload(name: str, device, mode: str, nb: int = B_CLIPS):
    """Returns (engine, output kind, roofline work dict, launches per step)."""
    precision = MODES[(name, mode)][0]
    from paper_1912_12055_b200 import banks
    from paper_1912_12055_b200.engine import CqtLongEngine, Cqt2010Engine, DftEngine
    from paper_1912_12055_b200.spectro import CqtConfig, cqt2010_plan

    if name in ("stft", "mel", "melpow2"):
        nf, _ = banks.frequency_scale("no", 2048, SR, 50.0, 6000.0, None)
        h_re, h_im = banks.dft_kernels(nf, banks.make_window("hann", 2048, True))
        eng = DftEngine(h_re, h_im, 512, precision=precision, device=device)
        kind = "magnitude"
        if name in ("mel", "melpow2"):
            w, _ = banks.mel_filter_bank(SR, 2048, 128, formula="slaney", norm="none")
            eng.set_mel(w, power=2.0 if name == "melpow2" else 1.0)
            kind = "mel"
        work = {"bound": "tensor", "per_batch": FLOP_STFT if name == "stft" else FLOP_MEL, "unit": "TFLOP/s",
                "kernel": "stft_gemm_kernel"}
        return eng, kind, work, 2
    if name == "cqt1992v2":
        cfg = CqtConfig(sr=SR)
        k, lens = banks.cqt_time_kernels(SR, cfg.bin_freqs_hz, 12, "hann", 1)
        eng = CqtLongEngine(k, 512, "reflect", precision=precision, device=device)
        work = {"bound": "tensor", "per_batch": 4.0 * M_FRAMES * float(lens.sum()), "unit": "TFLOP/s",
                "kernel": "cqt1992 hybrid (egemm + schedule)"}
        return eng, "magnitude", work, 2
    if name == "train":
        import torch.distributed as dist
        world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
        work = {"bound": "tensor", "per_batch": FLOP_TRAIN, "unit": "TFLOP/s",
                "kernel": "train step (stft_gemm fwd + rgemm dW/dS/dK + glue)"}
        return TrainStep(device, precision, world, nb, "tf32" if mode.endswith("onepass") else "split"), None, work, 0
    if name == "cqt2010v2":
        cfg = CqtConfig(sr=SR)
        p = cqt2010_plan(cfg)
        eng = Cqt2010Engine(p["taps"], p["top_kernels"], p["early_stages"], p["n_octaves"], p["kernel_hop"],
                            p["first_bin"], 12, 84, "reflect", device=device, precision=precision)
        work = {"bound": "hbm", "per_batch": float(BYTES_CQT2010), "unit": "GB/s",
                "kernel": "cqt2010v2 route (front + back end)"}
        return eng, "magnitude", work, 2 + (p["early_stages"] - 2) + 6 + 7
    raise ValueError(name)


L2_BYTES = 126 * 1024 * 1024
_flush_buf = None


def run_timed(eng, kind, x, steps, warmup, torch, stream, time_gemm=True, barrier=None, on_start=None):
    """W untimed steps then exactly K timed steps; events around each step and
    around the GEMM launch inside it (for the roofline).  When the input is
    smaller than 2x L2 (a rank's shard at N >= 4) a 256 MB buffer is written
    between steps, outside the step events, so no step reads a warm L2."""
    global _flush_buf
    staged = hasattr(eng, "stage") and time_gemm
    flush = x.numel() * 4 < 2 * L2_BYTES
    if flush and _flush_buf is None:
        _flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=x.device)
    for _ in range(warmup):
        eng.forward(x, kind)
    torch.cuda.synchronize()
    if barrier is not None:
        barrier()
    torch.cuda.synchronize()
    if on_start is not None:  # e.g. the clock sampler: the timed region starts here
        on_start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    g_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        if flush:
            _flush_buf.fill_(float(i))
        ev[i][0].record(stream)
        if staged:
            B, Ls = eng.stage(x)
            g_ev[i][0].record(stream)
            eng.run_staged(B, Ls, kind)
            g_ev[i][1].record(stream)
        else:
            eng.forward(x, kind)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    total = sum(a.elapsed_time(b) for a, b in ev)
    gemm = statistics.mean(a.elapsed_time(b) for a, b in g_ev) if staged else total / steps
    return total / steps, gemm


def _ref_module():
    """The unmodified reference package, installed (git-ignored) into baseline/_ref
    by `pip install --target baseline/_ref`; None if absent."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "spectro")):
        if p not in sys.path:
            sys.path.insert(0, p)
        import spectro
        return spectro
    return None


def reference_step_fn(name: str):
    """(per-clip callable, signal factory, kind, label) for the reference's own CPU
    path of `name`: banks built once here (init is outside the timed region, as
    the paper excludes it), clips mapped by the reference's
    `batch_transform` (transforms.py:370-388) with one BLAS thread per worker."""
    import numpy as np
    S = _ref_module()
    if S is not None:
        if name == "stft":
            tr = S.Stft(S.StftParams(n_fft=2048, hop_length=512, output="magnitude"), SR)
        elif name == "mel":
            tr = S.MelSpec(S.MelParams(n_fft=2048, n_mels=128, hop_length=512), SR)
        elif name == "cqt1992v2":
            tr = S.Cqt1992v2(S.CqtConfig(sr=SR))
        elif name == "cqt2010v2":
            tr = S.Cqt2010v2(S.CqtConfig(sr=SR))
        else:  # train: joint trainable STFT + Mel layer, forward + VJP per clip (gradients.py:103-149)
            scale = S.build_frequency_scale("no", 2048, SR)
            dft = S.build_dft_kernels(scale, S.make_window("hann", 2048, periodic=True))
            melb = S.build_mel_filter_bank(SR, 2048, 128, formula="slaney")
            stft_layer = S.TrainableLayer(dft, hop=512)
            mel_layer = S.TrainableLayer(melb, hop=512, stft_bank=dft)
            W = mel_layer.params()["weights"]
            g = np.full((128, T_FRAMES), 1e-3)

            def tr(x):
                gw = S.spectrogram_vjp(x, mel_layer, g)["weights"]
                gh = S.spectrogram_vjp(x, stft_layer, W.T @ g)
                return gw, gh["h_re"], gh["h_im"]
        return tr, (lambda row: S.Signal(row, SR)), "reference", (lambda sigs, threads: S.batch_transform(
            sigs, tr, threads=threads))
    # the oracle restatement (kind "port") when baseline/_ref was not installed
    from oracle import spectro_oracle as O
    h_re, h_im = O.stft_bank(2048, SR)
    W = O.mel_bank(SR, 2048, 128, formula="slaney")
    kern = O.cqt_time_bank(O.CqtCfg(sr=SR))[0] if name == "cqt1992v2" else None
    plan = O.cqt2010_plan(O.CqtCfg(sr=SR)) if name == "cqt2010v2" else None

    def train_clip(c):
        fr, re, im, Sm = O.smooth_mag_forward(c, h_re, h_im, 512)
        g = np.full((128, Sm.shape[1]), 1e-3)
        dW = g @ Sm.T
        dS = W.T @ g
        return dW, (dS * re / Sm) @ fr, (dS * im / Sm) @ fr

    fn = {
        "train": train_clip,
        "stft": lambda c: O.stft_clip(c, h_re, h_im, 512),
        "mel": lambda c: O.mel_clip(c, h_re, h_im, W, 512),
        "cqt1992v2": lambda c: O.cqt1992v2_clip(c, kern, 512),
        "cqt2010v2": lambda c: O.cqt2010v2_clip(c, O.CqtCfg(sr=SR), plan),
    }[name]

    def run(sigs, threads):
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as pool:
            return list(pool.map(fn, sigs))
    return fn, (lambda row: row), "port", run


def reference_clips(n: int):
    """The first n clips of the synthetic batch: N(0, 0.5^2) float32 (cli.py:98-99),
    float32-rounded then float64 as the reference sees them."""
    import numpy as np
    rng = np.random.default_rng(0)
    return (rng.standard_normal((n, L_SAMPLES), dtype=np.float32) * np.float32(0.5)).astype(np.float64)


def cpu_reference(name: str, max_seconds: float, threads: int):
    """CPU baseline leg of the GPU arm: the reference's batch_transform over a
    bounded sample of the batch (~max_seconds).  Returns (clips/s, clips, s, kind)."""
    _, mk, kind, run = reference_step_fn(name)
    pool = [mk(r) for r in reference_clips(max(threads, 1) * 2)]
    run(pool[:threads], threads)  # warm the pool / BLAS
    done, t0 = 0, time.perf_counter()
    while True:
        run(pool, threads)
        done += len(pool)
        el = time.perf_counter() - t0
        if el >= max_seconds or done >= B_CLIPS:
            break
    return done / el, done, el, kind


def reference_arm(args, threads: int, metric: str):
    """`bench.py --impl reference`: the reference's own CPU implementation of the
    workload, each step one batch_transform over a sample of the 1,770-clip batch
    (the whole batch when (K + W) full steps fit the time budget)."""
    _, mk, kind, run = reference_step_fn(args.workload)
    probe = [mk(r) for r in reference_clips(max(threads, 1) * 2)]
    run(probe[:threads], threads)
    t0 = time.perf_counter()
    run(probe, threads)
    per_clip = (time.perf_counter() - t0) / len(probe)
    n = int(args.ref_budget / max(1, args.steps + args.warmup) / per_clip)
    n = max(threads, min(B_CLIPS, n))
    sigs = [mk(r) for r in reference_clips(n)]
    for _ in range(args.warmup):
        run(sigs, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(sigs, threads)
    el = time.perf_counter() - t0
    v = n * args.steps / el
    src = ("spectro 0.1.0 (the reference, baseline/_ref), batch_transform" if kind == "reference"
           else "oracle restatement (baseline/_ref not installed)")
    sample = f"{n} of the 1,770 clips x 80,000 samples per step ({src}, {threads} threads x 1 BLAS thread)"
    return {
        "impl": "reference", "metric": metric, "value": v, "unit": "spectrograms/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * el / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0, 0.5^2) float32 clips (cli.py:98-99), as float64",
        "config": {"workload": WORKLOADS[args.workload], "clips_per_step": n, "samples": L_SAMPLES,
                   "threads": threads, "banks": "built once, outside the timed region"},
        "cpu_baseline": {"value": v, "unit": "spectrograms/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "spectrograms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def metric_name(workload: str) -> str:
    """One metric string for both arms (the driver divides only like by like)."""
    return f"{workload} spectrograms/s on the 1,770-clip x 80,000-sample batch"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="mel", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="f16", choices=["f16", "tf32", "fp32", "3xtf32", "tf32-onepass"],
                    help="operand mode (bench.MODES): f16 = the fastest <= 1e-3 mode, fp32 = the <= 1e-5 mode")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="seconds the reference arm may spend on its W + K steps")
    ap.add_argument("--no-breakdown", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    metric = metric_name(args.workload)

    if args.impl == "reference":
        if rank == 0:  # the reference is a CPU package: rank 0 alone runs it
            print(json.dumps(reference_arm(args, threads, metric)))
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) for the driver's log check
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device)
    hbm_peak, bf16_peak, peak_src = load_peaks()
    # TF32 tensor peak = half the measured dense bf16 peak (same MMA datapath, half the
    # K per instruction); the STFT GEMM can exceed it because the bf16 figure was
    # measured under the power cap at a lower SM clock (MEASURED_PEAKS.json clocks)
    tf32_peak = bf16_peak / 2.0
    traffic = load_traffic()

    # strong scaling: the 1,770-clip batch is sharded over the ranks (SURVEY.md section 8e:
    # 222, 222, 221 x 6 on 8 GPUs); forward needs no collective
    from paper_1912_12055_b200.dist import shard_range
    lo, hi = shard_range(B_CLIPS, rank, world)
    nb = hi - lo
    g = torch.Generator(device=device)
    g.manual_seed(1234)
    x_full = torch.randn(B_CLIPS, L_SAMPLES, device=device, generator=g) * 0.5
    x = x_full[lo:hi].contiguous()
    del x_full

    def roofline(work, kernel_ms, clips=B_CLIPS, mma="tf32"):
        t = kernel_ms / 1e3
        per = work["per_batch"] * clips / B_CLIPS
        if work["bound"] == "tensor":
            ach, peak = per / t / 1e12, (bf16_peak if mma == "f16" else tf32_peak)
        else:
            ach, peak = per / t / 1e9, hbm_peak
        return {"bound": work["bound"], "achieved": ach, "peak": peak, "unit": work["unit"], "frac": ach / peak,
                # measured per precision where a capture exists (kernel:workload:precision), else the
                # default mode's capture (kernel:workload)
                "traffic": (traffic.get(f'{work["kernel"]}:{args.workload}:{args.precision}',
                                        traffic.get(work["kernel"] + ":" + args.workload)) if work["kernel"] else None),
                "kernel": work["kernel"], "kernel_ms": kernel_ms,
                "peak_source": ((f"FP16 dense = measured bf16 {bf16_peak:.1f} TF/s ({peak_src}, burst)" if mma == "f16"
                                 else f"TF32 = measured dense bf16 {bf16_peak:.1f} TF/s / 2 ({peak_src}, burst)")
                                if work["bound"] == "tensor" else f"HBM copy {hbm_peak:.1f} GB/s ({peak_src})"),
                "work_per_step": per}

    from paper_1912_12055_b200 import _lib
    eng, kind, work, _ = build_workload(args.workload, device, args.precision, nb)
    staged = args.workload not in ("cqt2010v2", "train")

    clocks = Clocks(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = _lib.load().nnab_launch_count()
    ms, gemm_ms = run_timed(eng, kind, x, args.steps, args.warmup, torch, stream, time_gemm=staged,
                            barrier=(dist.barrier if world > 1 else None),
                            on_start=(clocks.start if rank == 0 else None))
    launches_total = _lib.load().nnab_launch_count() - n0  # includes the W warm-up steps
    launches = launches_total * args.steps // (args.steps + args.warmup)
    ck = clocks.stop() if rank == 0 else None
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = B_CLIPS / (ms / 1e3)  # whole-job clips / max-over-ranks step time
    mode = MODES[(args.workload, args.precision)] if (args.workload, args.precision) in MODES else None
    if mode is None:
        raise SystemExit(f"workload {args.workload} has no {args.precision} mode")
    rf = roofline(work, gemm_ms if staged else ms, nb, mode[2])

    # end to end through the C ABI host path: pinned input -> pinned output,
    # H2D + compute + D2H inside the timed region, chunked with copy/compute overlap
    e2e = None

    def e2e_time(fn, ks):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ks):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        et = e0.elapsed_time(e1) / ks
        if world > 1:
            t = torch.tensor([et], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        return et

    ks = max(3, min(10, args.steps))
    if args.workload in ("stft", "mel", "melpow2", "cqt1992v2", "cqt2010v2"):
        xh = x.cpu().pin_memory()
        out_rows = {"stft": 1025, "mel": 128, "melpow2": 128}.get(args.workload, 84)
        oh = torch.empty(nb, out_rows, T_FRAMES, dtype=torch.float32, pin_memory=True)
        chunk = 118 if args.workload in ("stft", "mel", "melpow2") else 148
        et = e2e_time(lambda: eng.forward_host(xh, kind, chunk_clips=chunk, out_host=oh), ks)
        path = {"cqt1992v2": "nnab_cqt1992v2_hybrid_forward_host", "cqt2010v2": "nnab_cqt2010v2_forward_host"}.get(
            args.workload, "nnab_stft_forward_host")
        e2e = {"value": B_CLIPS / (et / 1e3), "unit": "spectrograms/s", "ms_per_step": et,
               "h2d_bytes_per_step": nb * L_SAMPLES * 4, "d2h_bytes_per_step": nb * out_rows * T_FRAMES * 4,
               "path": path + " (C ABI, pinned host buffers, chunked H2D / compute / D2H on 3 streams)"}
        del xh, oh
    elif args.workload == "train":
        # pinned host batch -> device, fwd + bwd (+ all-reduce), kernel grads -> host, every
        # step; the H2D copy of step i+1 runs on a copy stream under step i's compute
        # (double-buffered device input, as a prefetching data loader would)
        xh = x.cpu().pin_memory()
        params = list(eng.m.parameters())
        gh = [torch.empty(p.shape, dtype=torch.float32, pin_memory=True) for p in params]
        xd = [torch.empty_like(x), torch.empty_like(x)]
        cs = torch.cuda.Stream(device)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]

        def issue_copy(i, after=None):
            b = i % 2
            if after is not None:
                cs.wait_event(after)
            cs.wait_event(free[b])  # step i-2 is done reading this buffer
            with torch.cuda.stream(cs):
                xd[b].copy_(xh, non_blocking=True)
            ready[b].record(cs)

        def e2e_steps(n, start_event=None):
            issue_copy(0, start_event)
            for i in range(n):
                b = i % 2
                stream.wait_event(ready[b])
                eng.forward(xd[b])
                free[b].record(stream)
                if i + 1 < n:
                    issue_copy(i + 1)
                for hbuf, p in zip(gh, params):
                    hbuf.copy_(p.grad, non_blocking=True)

        e2e_steps(2)
        torch.cuda.synchronize()
        k5 = max(3, min(5, args.steps))
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_steps(k5, e0)
        e1.record(stream)
        torch.cuda.synchronize()
        et = e0.elapsed_time(e1) / k5
        if world > 1:
            t = torch.tensor([et], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": B_CLIPS / (et / 1e3), "unit": "spectrograms/s", "ms_per_step": et,
               "h2d_bytes_per_step": nb * L_SAMPLES * 4,
               "d2h_bytes_per_step": int(sum(p.numel() for p in params) * 4),
               "path": "layers.MelSpectrogram(trainable_mel, trainable_STFT) fwd+bwd, pinned H2D input (next step's "
                       "copy overlapped on a second stream), D2H grads"}
        del xh, xd

    breakdown = {}
    if rank == 0 and world == 1 and not args.no_breakdown:
        for name in ["stft", "mel", "melpow2", "cqt1992v2", "cqt2010v2", "train"]:
            for prec in BREAKDOWN_MODES[name]:
                if name == args.workload and prec == args.precision:
                    continue
                e, k, w, _ = build_workload(name, device, prec, nb)
                st = name not in ("cqt2010v2", "train")
                m, gm = run_timed(e, k, x, 20 if name != "train" else 5, 3, torch, stream, time_gemm=st)
                r = roofline(w, gm if st else m, nb, MODES[(name, prec)][2])
                breakdown[f"{name}_{prec}"] = {"ms_per_step": m, "value": nb / (m / 1e3),
                                               "roofline_frac": r["frac"], "achieved": r["achieved"],
                                               "unit": r["unit"], "kernel_ms": r["kernel_ms"],
                                               "dtype": MODES[(name, prec)][1]}
                del e
        breakdown[f"{args.workload}_{args.precision}"] = {"ms_per_step": ms, "value": value,
                                                          "roofline_frac": rf["frac"], "achieved": rf["achieved"],
                                                          "unit": rf["unit"], "kernel_ms": rf["kernel_ms"]}

    cpu = None
    if rank == 0 and world == 1:
        v, n, el, kind_ref = cpu_reference(args.workload, args.cpu_seconds, threads)
        cpu = {"value": v, "unit": "spectrograms/s", "cores": threads, "kind": kind_ref,
               "sample": f"{n} clips x 80,000 samples ({el:.1f} s, "
                         + ("the reference spectro.batch_transform" if kind_ref == "reference"
                            else "oracle restatement") + f", {threads} threads x 1 BLAS thread)"}

    if rank == 0:
        line = {
            "metric": metric,
            "value": value, "unit": "spectrograms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": mode[1],
            "data": "synthetic: N(0, 0.5^2) float32 clips generated on device (cli.py:98-99 distribution)",
            "config": {"workload": WORKLOADS[args.workload], "global_clips": B_CLIPS, "clips_per_rank": nb,
                       "samples": L_SAMPLES, "sr": SR, "precision": args.precision,
                       "parallelism": f"dp{world}: the 1,770 clips sharded over ranks (dist.shard_range), "
                                      "no data-path collective" + ("; one gradient all-reduce per step"
                                                                   if args.workload == "train" else ""),
                       "l2": f"inputs {nb * L_SAMPLES * 4 / 1e6:.0f} MB per rank per step"
                             + (" > 126 MB L2 (no flush needed)" if nb * L_SAMPLES * 4 > 126e6 else
                                ", L2 flushed between steps")},
            "roofline": rf,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": ck,
            "transforms": breakdown or None,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
