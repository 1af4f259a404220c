import os, sys, subprocess, json
for st, wl in [("4", "stft"), ("3", "stft"), ("2", "stft"), ("3", "mel"), ("2", "mel")]:
    env = dict(os.environ, NNAB_DEBUG_STAGES=st)
    r = subprocess.run([sys.executable, "bench.py", "--workload", wl, "--steps", "30", "--warmup", "3", "--no-breakdown",
                        "--cpu-seconds", "0.1"], env=env, capture_output=True, text=True)
    lines = r.stdout.strip().splitlines()
    if not lines:
        print(st, wl, "FAILED", r.stderr[-300:]); continue
    d = json.loads(lines[-1])
    print(st, wl, "gemm ms", round(d["roofline"]["kernel_ms"], 3), "step ms", round(d["ms_per_step"], 3))
