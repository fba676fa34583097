"""C1 / C2 single-image rate per stage-kernel mode: auto (split kernel + ordered
reduction, 2 launches per stage) against the cluster kernel (modes 10 / 11,
one launch per stage) for each cluster size.  Usage: python tools/cluster_perf.py"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth


def rate(dm, f, out, work, n=30):
    for _ in range(5): dm.despeckle(f, out=out, work=work, check=False)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): dm.despeckle(f, out=out, work=work, check=False)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n)
    return best


for key, B in (("c2", 1), ("c1", 1), ("c2", 2), ("c3", 16)):
    cfg = synth.CONFIGS[key]
    model = synth.config_model(cfg)
    f = torch.from_numpy(np.stack([synth.noisy_image(cfg, i)[1] for i in range(B)])).cuda()
    dm = tn.device_model_for(model)
    out = torch.empty_like(f); work = torch.empty_like(f)
    px = B * cfg.H * cfg.W
    ref = None
    for label, mode, cl in (("auto", 0, 0), ("split_large", 6, 0), ("cluster_large cl=auto", 10, 0),
                            ("cluster_large cl=2", 10, 2), ("cluster_large cl=3", 10, 3),
                            ("cluster_large cl=4", 10, 4), ("cluster_large cl=6", 10, 6),
                            ("cluster_large cl=8", 10, 8),
                            ("cluster_small cl=auto", 11, 0), ("cluster_small cl=3", 11, 3),
                            ("cluster_small cl=6", 11, 6)):
        _lib.set_stage_kernel(mode); _lib.set_cluster_size(cl)
        try:
            ms = rate(dm, f, out, work)
            o = out.clone()
            if ref is None: ref = o
            err = float(((o - ref).abs() / ref.abs()).max())
            print(f"{key} B={B} {label:24s}: {ms*1e3:8.1f} us/despeckle {px/ms/1e3:8.1f} MPix/s  max rel diff vs auto {err:.2e}", flush=True)
        except Exception as e:
            print(f"{key} B={B} {label}: {type(e).__name__}: {e}", flush=True)
        finally:
            _lib.set_stage_kernel(0); _lib.set_cluster_size(0)
