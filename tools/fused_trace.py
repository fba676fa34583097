"""Per-CTA cycle accounting of the fused dataflow kernel (build with
-DTNRD_FUSED_TRACE, load through TNRD_LIB_PATH): total, waiting on
dependencies, reducing tiles, staging u + params, claims."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import _lib, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
model = synth.config_model(cfg)
f = torch.from_numpy(synth.noisy_image(cfg, 0)[1]).cuda()
dm = tn.device_model_for(model)
for _ in range(3):
    dm.despeckle(f)
torch.cuda.synchronize()
L = _lib.load()
buf = (ctypes.c_longlong * (4096 * 5))()
L.tnrd_debug_fused_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.tnrd_debug_fused_trace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.int64).reshape(4096, 5)
a = a[a[:, 0] > 0]
tot, wait, red, stg, n = a.T
print(f"{len(a)} CTAs; total cycles mean {tot.mean():.0f} max {tot.max()}; "
      f"wait {wait.sum() / tot.sum():.3f}, reduce {red.sum() / tot.sum():.3f}, "
      f"stage {stg.sum() / tot.sum():.3f} of CTA time; claims/CTA {n.mean():.1f}; "
      f"per-claim cycles {(tot.sum() / n.sum()):.0f}")
