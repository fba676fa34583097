"""Small despeckles through every stage-kernel variant (for compute-sanitizer
memcheck / racecheck runs; each tool in its own gpurun call)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import _lib, synth  # noqa: E402

modes = [int(m) for m in (sys.argv[1:] or ["3", "4", "2"])]
rng = np.random.default_rng(0)
for mode in modes:
    _lib.set_stage_kernel(mode)
    for m, (H, W) in ((7, (70, 90)), (5, (40, 33)), (9, (50, 60)), (3, (9, 200))):
        if mode == 2 and m == 9:
            continue
        model = synth.make_model(m, 20, 2, 63, seed=m)
        f = rng.uniform(0, 300, (H, W)).astype(np.float32)
        u, _ = tn.run_diffusion(f, model)
        assert np.all(np.isfinite(u)) and np.all(u > 0)
    print("mode", mode, "ok", flush=True)
