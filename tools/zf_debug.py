"""Debug the z-field stage: z planes vs a torch conv, one stage vs the
CUDA-core kernel."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import _lib, synth
m = int(sys.argv[1]) if len(sys.argv) > 1 else 7
nk = int(sys.argv[2]) if len(sys.argv) > 2 else 8
H, W = 40, 70
model = synth.make_model(m, nk, 1, 63, seed=3)
f = torch.from_numpy(np.random.default_rng(1).uniform(1, 300, (H, W)).astype(np.float32)).cuda()
dm = tn.device_model_for(model)
_lib.set_stage_kernel(1)
ref = dm.despeckle(f)
torch.cuda.synchronize()
_lib.set_stage_kernel(8)
try:
    got = dm.despeckle(f)
    torch.cuda.synchronize()
    d = (got - ref).abs() / ref.abs()
    print("max rel diff vs cuda-core", d.max().item(), "argmax", np.unravel_index(d.argmax().item(), d.shape))
except Exception as e:
    print("ERR", e)
