"""One rank of the CPU (gloo) row-strip test: despeckles its strip with the
float64 oracle as the stage operator and the real halo exchange, then
writes its rows to an .npy file.  Launched by tests/test_strips_cpu.py."""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1702_07482_b200 import _lib, strips, synth  # noqa: E402


def oracle_stage_fn(a):
    def fn(t, u_in, f, u_out, layout, flags):
        h, n = layout.halo, layout.n
        lo = 0 if layout.has_top else h
        hi = n + 2 * h if layout.has_bottom else n + h
        u = u_in[lo:hi].numpy()
        if flags & _lib.STAGE_FLOOR_INPUT:
            u = np.maximum(u, 1e-6)
        out = O.stage(u, f[lo:hi].numpy(), a["kernels"][t], a["weights"][t],
                      a["centers"], a["gamma"], a["lams"][t])
        u_out[h:h + n] = torch.from_numpy(out[h - lo:h - lo + n])
    return fn


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--world", type=int)
    ap.add_argument("--port", type=int)
    ap.add_argument("--out")
    ap.add_argument("--H", type=int, default=61)
    ap.add_argument("--W", type=int, default=45)
    ap.add_argument("--m", type=int, default=7)
    a = ap.parse_args()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(a.port))
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    O.set_threads(1)
    model = synth.make_model(a.m, 5, 3, 63, seed=11)
    f = np.random.default_rng(3).uniform(0, 255, (a.H, a.W))
    lay = strips.StripLayout(a.H, a.W, a.world, a.rank, halo=a.m - 1)
    r0, r1 = lay.rows
    h = lay.halo
    f_ext = torch.zeros(lay.n + 2 * h, a.W, dtype=torch.float64)
    f_ext[h:h + lay.n] = torch.from_numpy(f[r0:r1])
    bufs = [torch.zeros_like(f_ext), torch.zeros_like(f_ext)]
    res = strips.run_strip(f_ext, oracle_stage_fn(O.model_arrays(model)),
                           model.num_stages, lay, bufs)
    np.save(a.out, res[h:h + lay.n].numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
