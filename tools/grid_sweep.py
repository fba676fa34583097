"""Despeckle rate vs grid size for each CUDA-core stage kernel: tile kernel
(mode 4), split kernel (6) and the cluster kernel (10) with 2 / 4 / 8 CTAs per
cluster -- the data behind the auto choice (cc_variant, tnrd_capi.cu).
Usage: python tools/grid_sweep.py [c3|c5]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = synth.CONFIGS[key]
model = synth.config_model(cfg)
dm = tn.device_model_for(model)
nb = 16 if key == "c3" else 4
base = torch.from_numpy(synth.noisy_batch(cfg, range(nb))).cuda()
Bs = [1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32, 64] if key == "c3" else [1, 2, 3, 4, 8]
MODES = (("auto", 0, 0), ("tile", 4, 0), ("split", 6, 0), ("cl2", 10, 2), ("cl3", 10, 3), ("cl4", 10, 4), ("cl8", 10, 8))
print(f"{key}: MPix/s per mode; tiles = B x {((cfg.H + 63) // 64) * ((cfg.W + 63) // 64)}")
print("   B " + " ".join(f"{m[0]:>8s}" for m in MODES))
for B in Bs:
    f = base.repeat((B + nb - 1) // nb, 1, 1)[:B].contiguous()
    out = torch.empty_like(f); work = torch.empty_like(f)
    px = B * cfg.H * cfg.W
    row = []
    for label, mode, cl in MODES:
        _lib.set_stage_kernel(mode); _lib.set_cluster_size(cl)
        try:
            for _ in range(3): dm.despeckle(f, out=out, work=work, check=False)
            torch.cuda.synchronize()
            n = max(3, 60 // B)
            best = 1e9
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(n): dm.despeckle(f, out=out, work=work, check=False)
                e1.record(); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / n)
            row.append(px / best / 1e3)
        except Exception as e:
            row.append(float("nan"))
        finally:
            _lib.set_stage_kernel(0); _lib.set_cluster_size(0)
    print(f"{B:4d} " + " ".join(f"{v:8.1f}" for v in row), flush=True)
