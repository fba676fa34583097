"""Gradient path throughput: loss_and_gradients of one
256x256 sample through all T = 5 stages of a C2-shaped model (7x7, Nk=48,
M=63), GPU (this package) or the reference's float64 numpy path (--ref, run
in the build container where /root/reference exists).  One JSON line."""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
ref = "--ref" in sys.argv
N = 256
if ref:
    sys.path.insert(0, "/root/reference/pkg/src")
    from specklediff import training as tr  # noqa: E402
    from specklediff.speckle import NoisyPair, SpeckleConfig  # noqa: E402
    sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
    from make_golden import ref_model  # noqa: E402
    model = ref_model(7, 48, 5, 63, seed=2)
else:
    from paper_1702_07482_b200 import synth  # noqa: E402
    from paper_1702_07482_b200 import training as tr  # noqa: E402
    from paper_1702_07482_b200.speckle import NoisyPair, SpeckleConfig  # noqa: E402
    model = synth.make_model(7, 48, 5, 63, seed=2)
rng = np.random.default_rng(0)
clean = rng.uniform(20, 235, (N, N))
noisy = clean * np.sqrt(rng.gamma(4.0, 0.25, (N, N)))
pair = NoisyPair(clean=clean, noisy=noisy, config=SpeckleConfig(4, 7))
reps = 1 if ref else 5
tr.loss_and_gradients(model, [pair], list(range(5)), 4)   # warm-up (GPU: model upload, JIT-free)
if not ref:
    import torch
    torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    total, acc = tr.loss_and_gradients(model, [pair], list(range(5)), 4)
dt = (time.perf_counter() - t0) / reps
print(json.dumps({"path": "reference numpy float64" if ref else "GPU tnrd_stage_backward",
                  "workload": f"loss_and_gradients, 1 sample {N}x{N}, T=5, 7x7, Nk=48, M=63",
                  "seconds": dt, "mpix_per_s": N * N / dt / 1e6,
                  "threads": os.cpu_count() if ref else None,
                  "loss": total}))
