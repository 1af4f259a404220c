#!/usr/bin/env python
"""Benchmark: spectrograms/s on the 1,770-clip x 80,000-sample batch (44.1 kHz)
plus the roofline fraction of the dominant kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload mel|stft|cqt1992v2|cqt2010v2|train]
    python bench.py --impl reference ...     # the reference's CPU path (oracle port) on the host cores

A step is one pass of the workload over one full batch already resident in
HBM (566 MB of input > 126 MB L2, so no L2 flush is needed between steps).
Multi-GPU: one process per GPU (torchrun); every rank processes its own full
batch (weak scaling, clips shard with no collective on the forward path);
`value` = all ranks' clips / max-over-ranks time.  Rank 0 prints ONE JSON line.
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
    "cqt1992v2": "CQT1992v2 84 bins 12/oct fmin=32.70 hop=512, magnitude (BASELINE config 3)",
    "cqt2010v2": "CQT2010v2 84 bins 12/oct fmin=32.70 hop=512 early downsample, magnitude (BASELINE config 4)",
    "train": "trainable STFT+Mel (trainable_mel + trainable_STFT, n_fft=2048 n_mels=128 hop=512) forward + "
             "backward (dW, dS, dh) + NCCL kernel-grad all-reduce (BASELINE config 5)",
}
FLOP_TRAIN = FLOP_MEL + 2.0 * M_FRAMES * 2048 * 2050 + 2 * (2.0 * M_FRAMES * 1025 * 128)  # 4.886e12 (section 8d)


class TrainStep:
    """One optimisation step's compute for config 5: forward of the trainable
    Mel layer, backward for the mel weights and both DFT banks, and (N > 1)
    the single flattened gradient all-reduce."""

    def __init__(self, device, precision, world):
        import torch
        from paper_1912_12055_b200.layers import MelSpectrogram
        self.m = MelSpectrogram(sr=SR, n_fft=2048, n_mels=128, hop_length=512, trainable_mel=True,
                                trainable_STFT=True, precision=precision, device=device)
        self.world = world
        gen = torch.Generator(device=device)
        gen.manual_seed(77)
        self.g = torch.randn(B_CLIPS, 128, T_FRAMES, device=device, generator=gen) * 1e-3

    def forward(self, x, kind=None):
        from paper_1912_12055_b200.dist import allreduce_grads
        for p in self.m.parameters():
            p.grad = None
        out = self.m(x)
        out.backward(self.g)
        if self.world > 1:
            allreduce_grads(list(self.m.parameters()))
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
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.path = index, None, f"/tmp/nnab_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
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
                for n, v in zip(names, parts[2:]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        note = None
        if not sm:  # timed region shorter than nvidia-smi's first sample: one query right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout
                parts = [p.strip() for p in out.strip().split(",")]
                sm.append(float(parts[0]))
                mx = float(parts[1])
                for n, v in zip(names, parts[2:]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
                note = "timed region shorter than the 100 ms sampler: one sample right after it"
            except Exception:
                return None
        d = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if note:
            d["note"] = note
        return d


# ------------------------------------------------------------------ workloads
def build_workload(name: str, device, precision: str):
    """Returns (step_fn, gemm_fn or None, launches_per_step, roofline dict builder, e2e fn)."""
    from paper_1912_12055_b200 import banks
    from paper_1912_12055_b200.engine import CqtLongEngine, Cqt2010Engine, DftEngine
    from paper_1912_12055_b200.spectro import CqtConfig, cqt2010_plan

    if name in ("stft", "mel"):
        nf, _ = banks.frequency_scale("no", 2048, SR, 50.0, 6000.0, None)
        h_re, h_im = banks.dft_kernels(nf, banks.make_window("hann", 2048, True))
        eng = DftEngine(h_re, h_im, 512, precision=precision, device=device)
        kind = "magnitude"
        if name == "mel":
            w, _ = banks.mel_filter_bank(SR, 2048, 128, formula="slaney", norm="none")
            eng.set_mel(w, power=1.0)
            kind = "mel"
        work = {"bound": "tensor", "per_batch": FLOP_MEL if name == "mel" else FLOP_STFT, "unit": "TFLOP/s",
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
        return TrainStep(device, precision, world), None, work, 0
    if name == "cqt2010v2":
        cfg = CqtConfig(sr=SR)
        p = cqt2010_plan(cfg)
        eng = Cqt2010Engine(p["taps"], p["top_kernels"], p["early_stages"], p["n_octaves"], p["kernel_hop"],
                            p["first_bin"], 12, 84, "reflect", device=device, precision=precision)
        work = {"bound": "hbm", "per_batch": float(BYTES_CQT2010), "unit": "GB/s", "kernel": "cqt2010v2 chain"}
        return eng, "magnitude", work, 2 + (p["early_stages"] - 2) + 6 + 7
    raise ValueError(name)


def run_timed(eng, kind, x, steps, warmup, torch, stream, time_gemm=True):
    """W untimed steps then exactly K timed steps; events around the whole step
    and around the GEMM launch inside it (for the roofline)."""
    staged = hasattr(eng, "stage") and time_gemm
    for _ in range(warmup):
        eng.forward(x, kind)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    g_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    ev0.record(stream)
    for i in range(steps):
        if staged:
            B, Ls = eng.stage(x)
            g_ev[i][0].record(stream)
            eng.run_staged(B, Ls, kind)
            g_ev[i][1].record(stream)
        else:
            eng.forward(x, kind)
    ev1.record(stream)
    torch.cuda.synchronize()
    total = ev0.elapsed_time(ev1)
    gemm = statistics.mean(a.elapsed_time(b) for a, b in g_ev) if staged else total / steps
    return total / steps, gemm


def cpu_reference(name: str, max_seconds: float, threads: int, min_clips: int | None = None):
    """The reference's CPU path restated by the oracle (kind 'port'), mapped over
    clips with a thread pool and one BLAS thread each (transforms.py:370-388)."""
    import numpy as np

    from oracle import spectro_oracle as O
    h_re, h_im = O.stft_bank(2048, SR)
    W = O.mel_bank(SR, 2048, 128, formula="slaney")
    kern = O.cqt_time_bank(O.CqtCfg(sr=SR))[0] if name == "cqt1992v2" else None
    plan = O.cqt2010_plan(O.CqtCfg(sr=SR)) if name == "cqt2010v2" else None
    def train_clip(c):  # joint trainable STFT + Mel layer: forward + vjp (gradients.py:61-129)
        fr, re, im, S = O.smooth_mag_forward(c, h_re, h_im, 512)
        g = np.ones((128, S.shape[1]))
        dW = g @ S.T
        dS = W.T @ g
        return (dS * re / S) @ fr + (dS * im / S) @ fr + dW.sum()

    fn = {
        "train": train_clip,
        "stft": lambda c: O.stft_clip(c, h_re, h_im, 512),
        "mel": lambda c: O.mel_clip(c, h_re, h_im, W, 512),
        "cqt1992v2": lambda c: O.cqt1992v2_clip(c, kern, 512),
        "cqt2010v2": lambda c: O.cqt2010v2_clip(c, O.CqtCfg(sr=SR), plan),
    }[name]
    rng = np.random.default_rng(0)
    chunk = max(threads, 1) * 2
    pool = (rng.standard_normal((chunk, L_SAMPLES)) * 0.5).astype(np.float32).astype(np.float64)
    done, t0 = 0, time.perf_counter()
    while True:
        O.map_clips(fn, pool, threads=threads)
        done += chunk
        el = time.perf_counter() - t0
        if el >= max_seconds or done >= B_CLIPS or (min_clips and done >= min_clips):
            break
    return done / el, done, el


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="mel", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-breakdown", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        # warm-up steps then K timed steps, each a bounded sample of the workload
        for _ in range(args.warmup):
            cpu_reference(args.workload, 0.0, threads, min_clips=1)
        t0 = time.perf_counter()
        clips = 0
        for _ in range(args.steps):
            _, n, _ = cpu_reference(args.workload, 0.0, threads, min_clips=1)
            clips += n
        el = time.perf_counter() - t0
        v = clips / el
        print(json.dumps({
            "impl": "reference", "metric": f"{args.workload} spectrograms/s (1,770-clip batch config)",
            "value": v, "unit": "spectrograms/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * el / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic N(0, 0.5^2) clips, float32-rounded",
            "config": {"workload": WORKLOADS[args.workload], "clips_per_step": 2 * threads, "samples": L_SAMPLES},
            "cpu_baseline": {"value": v, "unit": "spectrograms/s", "cores": threads, "kind": "port",
                             "sample": f"{2 * threads} clips x 80,000 samples per step"},
            "e2e": {"value": v, "unit": "spectrograms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device)
    hbm_peak, bf16_peak, peak_src = load_peaks()
    # no measured TF32 figure exists (MEASURED_PEAKS.json has bf16 only): the B200
    # profiling recipe's stated dense TF32 peak, 1.1 PFLOP/s (bf16/2 of the measured
    # cuBLAS number would be 820, which the STFT kernel already exceeds)
    tf32_peak = 1100.0
    traffic = load_traffic()

    g = torch.Generator(device=device)
    g.manual_seed(1234 + rank)
    x = torch.randn(B_CLIPS, L_SAMPLES, device=device, generator=g) * 0.5

    def roofline(work, t_ms, kernel_ms):
        t = kernel_ms / 1e3
        if work["bound"] == "tensor":
            ach = work["per_batch"] / t / 1e12
            peak = tf32_peak
        else:
            ach = work["per_batch"] / t / 1e9
            peak = hbm_peak
        return {"bound": work["bound"], "achieved": ach, "peak": peak, "unit": work["unit"], "frac": ach / peak,
                "traffic": traffic.get(work["kernel"] + ":" + args.workload) if work["kernel"] else None,
                "kernel": work["kernel"], "kernel_ms": kernel_ms,
                "peak_source": ("TF32 dense 1.1 PFLOP/s (B200_PROFILING.md fallback; no measured TF32 peak)"
                                if work["bound"] == "tensor" else f"HBM copy {peak_src}")}

    from paper_1912_12055_b200 import _lib
    eng, kind, work, _ = build_workload(args.workload, device, args.precision)
    staged = args.workload not in ("cqt2010v2", "train")

    clocks = Clocks(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if rank == 0:
        clocks.start()
    n0 = _lib.load().nnab_launch_count()
    ms, gemm_ms = run_timed(eng, kind, x, args.steps, args.warmup, torch, stream, time_gemm=staged)
    launches_total = _lib.load().nnab_launch_count() - n0  # includes the W warm-up steps
    launches = launches_total * args.steps // (args.steps + args.warmup)
    ck = clocks.stop() if rank == 0 else None
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = world * B_CLIPS / (ms / 1e3)
    rf = roofline(work, ms, gemm_ms if staged else ms)

    # end to end through the C ABI host path: pinned input -> pinned output,
    # H2D + compute + D2H inside the timed region, chunked with copy/compute overlap
    e2e = None
    if args.workload in ("stft", "mel"):
        xh = x.cpu().pin_memory()
        out_rows = 128 if kind == "mel" else 1025
        oh = torch.empty(B_CLIPS, out_rows, T_FRAMES, dtype=torch.float32, pin_memory=True)
        for _ in range(2):
            eng.forward_host(xh, kind, chunk_clips=118, out_host=oh)
        torch.cuda.synchronize()
        ks = max(3, min(10, args.steps))
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ks):
            eng.forward_host(xh, kind, chunk_clips=118, out_host=oh)
        e1.record(stream)
        torch.cuda.synchronize()
        et = e0.elapsed_time(e1) / ks
        if world > 1:
            t = torch.tensor([et], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": world * B_CLIPS / (et / 1e3), "unit": "spectrograms/s", "ms_per_step": et,
               "h2d_bytes_per_step": B_CLIPS * L_SAMPLES * 4, "d2h_bytes_per_step": B_CLIPS * out_rows * T_FRAMES * 4,
               "path": "nnab_stft_forward_host (C ABI, pinned host buffers, 15 chunks, 3-stream overlap)"}
        del xh, oh
    elif args.workload in ("cqt1992v2", "cqt2010v2"):
        # pinned host batch -> C ABI host entry (chunked H2D / compute / D2H) -> pinned host result
        xh = x.cpu().pin_memory()
        oh = torch.empty(B_CLIPS, 84, T_FRAMES, dtype=torch.float32, pin_memory=True)
        for _ in range(2):
            eng.forward_host(xh, kind, chunk_clips=148, out_host=oh)
        torch.cuda.synchronize()
        ks = max(3, min(10, args.steps))
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ks):
            eng.forward_host(xh, kind, chunk_clips=148, out_host=oh)
        e1.record(stream)
        torch.cuda.synchronize()
        et = e0.elapsed_time(e1) / ks
        if world > 1:
            t = torch.tensor([et], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": world * B_CLIPS / (et / 1e3), "unit": "spectrograms/s", "ms_per_step": et,
               "h2d_bytes_per_step": B_CLIPS * L_SAMPLES * 4, "d2h_bytes_per_step": B_CLIPS * 84 * T_FRAMES * 4,
               "path": ("nnab_cqt1992v2_hybrid_forward_host" if args.workload == "cqt1992v2" else
                        "nnab_cqt2010v2_forward_host") + " (C ABI, pinned host buffers, 12 chunks, 3-stream overlap)"}
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
        ks = max(3, min(5, args.steps))
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_steps(ks, e0)
        e1.record(stream)
        torch.cuda.synchronize()
        et = e0.elapsed_time(e1) / ks
        if world > 1:
            t = torch.tensor([et], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": world * B_CLIPS / (et / 1e3), "unit": "spectrograms/s", "ms_per_step": et,
               "h2d_bytes_per_step": B_CLIPS * L_SAMPLES * 4,
               "d2h_bytes_per_step": int(sum(p.numel() for p in params) * 4),
               "path": "layers.MelSpectrogram(trainable_mel, trainable_STFT) fwd+bwd, pinned H2D input (next step's "
                       "copy overlapped on a second stream), D2H grads"}
        del xh, xd

    breakdown = {}
    if rank == 0 and world == 1 and not args.no_breakdown:
        for name in ["stft", "mel", "cqt1992v2", "cqt2010v2", "train"]:
            for prec in ["tf32", "fp32"]:
                if name == args.workload and prec == args.precision:
                    continue
                e, k, w, _ = build_workload(name, device, prec)
                st = name not in ("cqt2010v2", "train")
                m, gm = run_timed(e, k, x, 20 if name != "train" else 5, 3, torch, stream, time_gemm=st)
                r = roofline(w, m, gm if st else m)
                breakdown[f"{name}_{prec}"] = {"ms_per_step": m, "value": B_CLIPS / (m / 1e3),
                                               "roofline_frac": r["frac"], "achieved": r["achieved"],
                                               "unit": r["unit"], "kernel_ms": r["kernel_ms"]}
                del e
        breakdown[f"{args.workload}_{args.precision}"] = {"ms_per_step": ms, "value": value / world,
                                                          "roofline_frac": rf["frac"], "achieved": rf["achieved"],
                                                          "unit": rf["unit"], "kernel_ms": rf["kernel_ms"]}

    cpu = None
    if rank == 0 and world == 1:
        v, n, el = cpu_reference(args.workload, args.cpu_seconds, threads)
        cpu = {"value": v, "unit": "spectrograms/s", "cores": threads, "kind": "port",
               "sample": f"{n} clips x 80,000 samples ({el:.1f} s, oracle restatement, {threads} threads x 1 BLAS thread)"}

    if rank == 0:
        line = {
            "metric": f"{args.workload} spectrograms/s on the 1,770-clip batch (+ roofline fraction)",
            "value": value, "unit": "spectrograms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": (("f16 operands (exact per-clip power-of-two scale), f32 accumulate" if args.precision == "tf32"
                       else "f32 (CUDA cores)") if args.workload == "cqt2010v2"
                      else "tf32" if args.precision == "tf32" else "3xtf32"),
            "data": "synthetic: N(0, 0.5^2) float32 clips generated on device (cli.py:98-99 distribution)",
            "config": {"workload": WORKLOADS[args.workload], "clips_per_gpu": B_CLIPS, "global_clips": B_CLIPS * world,
                       "samples": L_SAMPLES, "sr": SR, "precision": args.precision,
                       "parallelism": f"dp{world}: clips sharded per rank, no data-path collective",
                       "l2": "inputs 566 MB per step > 126 MB L2 (no flush needed)"},
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
