"""Run a few despeckles of a workload subset (for ncu captures)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import synth
key = sys.argv[1] if len(sys.argv) > 1 else "c3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = synth.CONFIGS[key]
model = synth.config_model(cfg)
if cfg.tiled:
    f = torch.from_numpy(np.ascontiguousarray(synth.scene_crop(cfg, 0, cfg.H, 0, cfg.W), dtype=np.float32)).cuda()
else:
    f = torch.from_numpy(np.stack([synth.noisy_image(cfg, i)[1] for i in range(B)])).cuda()
dm = tn.device_model_for(model)
for _ in range(3):
    dm.despeckle(f)
torch.cuda.synchronize()
print("ok")
