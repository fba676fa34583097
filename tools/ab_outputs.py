"""Run fixed inputs through the library at TNRD_LIB_PATH and save the
outputs (A/B bit-identity checks between builds).  Usage:
    TNRD_LIB_PATH=... python tools/ab_outputs.py <out.npz>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import _lib, synth  # noqa: E402

out = {}
rng = np.random.default_rng(0)
cases = {
    "c2": (synth.config_model(synth.CONFIGS["c2"]), synth.noisy_batch(synth.CONFIGS["c2"], [0])[0]),
    "c3x16": (synth.config_model(synth.CONFIGS["c3"]), synth.noisy_batch(synth.CONFIGS["c3"], range(16))),
    "c1": (synth.config_model(synth.CONFIGS["c1"]), synth.noisy_batch(synth.CONFIGS["c1"], [0])[0]),
    "m3": (synth.make_model(3, 10, 2, 63, seed=4), rng.uniform(1, 255, (8, 300, 260)).astype(np.float32)),
    "m5": (synth.make_model(5, 13, 2, 63, seed=5), rng.uniform(1, 255, (8, 260, 300)).astype(np.float32)),
    "c5x2": (synth.config_model(synth.CONFIGS["c5"]), synth.noisy_batch(synth.CONFIGS["c5"], range(2))),
    # tile-aligned shapes: every image edge is a tile edge (EDGE backward variants)
    "m3a": (synth.make_model(3, 10, 2, 63, seed=4), rng.uniform(1, 255, (3, 128, 192)).astype(np.float32)),
    "m5a": (synth.make_model(5, 13, 2, 63, seed=5), rng.uniform(1, 255, (2, 64, 64)).astype(np.float32)),
    "m9a": (synth.make_model(9, 6, 2, 63, seed=6), rng.uniform(1, 255, (192, 64)).astype(np.float32)),
}
for mode in (_lib.KERNEL_AUTO, _lib.KERNEL_SMALL_TILES, _lib.KERNEL_LARGE_TILES, _lib.KERNEL_SPLIT_LARGE,
             _lib.KERNEL_CLUSTER_LARGE, _lib.KERNEL_CLUSTER_SMALL):
    _lib.set_stage_kernel(mode)
    for k, (model, f) in cases.items():
        dm = tn.device_model_for(model)
        u = dm.despeckle(torch.from_numpy(f).cuda()).cpu().numpy()
        out[f"{k}_mode{mode}"] = u
_lib.set_stage_kernel(_lib.KERNEL_AUTO)
np.savez(sys.argv[1], **out)
print("saved", len(out))
