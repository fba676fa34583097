"""C3-model despeckle rate vs batch size through tnrd_despeckle (auto mode:
tile kernel + batch fork), CUDA events, with nvidia-smi clocks / power
sampled during each timed block.  Usage: [TNRD_LIB_PATH=...] python tools/batch_perf.py"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
model = synth.config_model(cfg)
dm = tn.device_model_for(model)
base = torch.from_numpy(synth.noisy_batch(cfg, range(16))).cuda()
for B in ([16, 64, 256] if cfg.name == "c3" else [4, 16, 32]):
    f = base.repeat((B + 15) // 16, 1, 1)[:B].contiguous()
    out = torch.empty_like(f)
    work = torch.empty_like(f)
    for _ in range(3):
        dm.despeckle(f, out=out, work=work, check=False)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    n = max(3, int(2000 // B))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        dm.despeckle(f, out=out, work=work, check=False)
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    s = smi.communicate()[0].strip().splitlines()
    clk = [float(x.split(",")[0]) for x in s if x.count(",") == 1]
    pw = [float(x.split(",")[1]) for x in s if x.count(",") == 1]
    ms = e0.elapsed_time(e1) / n
    px = B * cfg.H * cfg.W
    print(f"{cfg.name} B={B:4d}: {ms:8.3f} ms/despeckle {px / ms / 1e3:7.1f} MPix/s  "
          f"sm_mhz median {np.median(clk):.0f} min {min(clk):.0f}  power median {np.median(pw):.0f} W", flush=True)
