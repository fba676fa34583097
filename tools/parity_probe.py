"""Parity of the GPU path against the CPU oracle on full C1 / C2 images, with
each tap source / RBF table (tnrd_set_param_taps): max relative error and
|delta PSNR| (the north_star bars are 1e-4 and 0.01 dB)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import _lib, synth  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)


def psnr(u, clean):
    mse = np.mean((np.asarray(u, np.float64) - clean) ** 2)
    return 10 * np.log10(255.0 ** 2 / mse)


for key in ("c1", "c2"):
    cfg = synth.CONFIGS[key]
    model = synth.config_model(cfg)
    clean, f = synth.noisy_image(cfg, 0)
    ref = O.run_diffusion(f.astype(np.float64), model)
    for pt in (True, False):
        _lib.set_param_taps(pt)
        u, _ = tn.run_diffusion(f, model)
        rel = float(np.max(np.abs(u - ref) / np.abs(ref)))
        dp = abs(psnr(u, clean) - psnr(ref, clean))
        print(f"{key} param_taps={int(pt)} (RBF {'cubic' if pt else 'degree 7'}): "
              f"max rel err {rel:.2e}  |dPSNR| {dp:.2e} dB", flush=True)
_lib.set_param_taps(True)
