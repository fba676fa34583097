import sys, time, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import synth
for key, B in (("c2", 1), ("c3", 16), ("c5", 4), ("c1", 1)):
    cfg = synth.CONFIGS[key]
    model = synth.config_model(cfg)
    f = torch.from_numpy(np.stack([synth.noisy_image(cfg, i)[1] for i in range(B)])).cuda()
    dm = tn.device_model_for(model)
    out = torch.empty_like(f); work = torch.empty_like(f)
    try:
        for _ in range(3): dm.despeckle(f, out=out, work=work, check=False)
    except NotImplementedError as e:
        print(f"{key}: {e}", flush=True)
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n): dm.despeckle(f, out=out, work=work, check=False)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    px = B * cfg.H * cfg.W
    print(f"{key} B={B}: {ms:.3f} ms/despeckle, {px/ms/1e3:.1f} MPix/s, {px*cfg.T/ms/1e3:.1f} MPix*st/s", flush=True)
