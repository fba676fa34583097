import glob
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_sessionfinish(session, exitstatus):
    """Debug bounds build (-DTNRD_BOUNDS, tools/bounds_run.sh): after the
    suite, the library's violation counters must be zero."""
    try:
        from paper_1702_07482_b200 import _lib
        L = _lib._lib
        if L is None or not hasattr(L, "tnrd_bounds_failures"):
            return
        import ctypes
        out = (ctypes.c_uint * 4)()
        L.tnrd_bounds_failures.restype = ctypes.c_int
        rc = L.tnrd_bounds_failures(out)
        line = (f"TNRD_BOUNDS: rc {rc}, {out[0]} violations"
                + (f" (first: kind {out[1]}, value {out[2]}, limit {out[3]})" if out[0] else ""))
        print("\n" + line)
        path = os.environ.get("TNRD_BOUNDS_REPORT")
        if path:
            with open(path, "a") as fh:
                fh.write(line + "\n")
        if rc != 0 or out[0]:
            session.exitstatus = 1
    except Exception as e:  # never mask the suite's own result
        print(f"\nTNRD_BOUNDS: report failed: {e}")


def golden_names(full_only=False):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        name = os.path.basename(p)[:-4]
        with np.load(p) as d:
            if "full" not in d.files:
                continue
            if full_only and not bool(d["full"]):
                continue
        out.append(name)
    return out


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as d:
        return {k: d[k] for k in d.files}


def golden_model(g, pkg=None):
    """Rebuild the golden case's model with OUR package's containers."""
    if pkg is None:
        import paper_1702_07482_b200 as pkg
    bw = float(g["rbf_bandwidth"])
    grid = pkg.RbfGrid(int(g["rbf_count"]), float(g["rbf_radius"]),
                       None if np.isnan(bw) else bw)
    stages = [pkg.StageParams(beta=float(b), coeffs=c, weights=w)
              for b, c, w in zip(g["betas"], g["coeffs"], g["weights"])]
    variant = str(g["variant"]) if "variant" in g else "prox"
    floor = float(g["floor"]) if "floor" in g else 1.0
    return pkg.DiffusionModel(stages=stages, filter_size=int(g["m"]), looks=1,
                              rbf=grid, variant=variant, floor=floor)


def parity_stats(u, ref, clean=None):
    """max relative error over non-degenerate pixels + max abs error on the
    degenerate ones (u_ref < 1e-6: the reference's naive prox loses all
    relative precision there, speckle.py:119-121) + PSNR delta."""
    u = np.asarray(u, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nd = np.abs(ref) >= 1e-6
    rel = float(np.max(np.abs(u[nd] - ref[nd]) / np.abs(ref[nd]))) if nd.any() else 0.0
    abs_deg = float(np.max(np.abs(u[~nd] - ref[~nd]))) if (~nd).any() else 0.0
    out = dict(rel=rel, abs_degenerate=abs_deg)
    if clean is not None:
        from oracle import oracle as O
        out["dpsnr"] = abs(O.psnr(u, clean, 255.0) - O.psnr(ref, clean, 255.0))
    return out


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
