"""Per-rank shard timing for the batch configs under each stage-kernel mode.

For N = 1, 2, 4, 8 a rank of `bench.py --gpus N` despeckles 256/N (C3) or
32/N (C5) images; this times one such shard on one GPU with the kernel
choice forced (4 = tile kernel, large tiles; 6 = split kernel, large tiles)
and with auto (0), so the auto heuristic can be checked against the wave
quantisation of the tile kernel on small shards.

C4 (one 16384^2 scene in row strips): a rank of N > 1 owns 16384/N rows and
reads m - 1 = 6 halo rows per internal edge; the proxy timed here is a
despeckle of a (16384/N + 12) x 16384 image (auto mode), i.e. the rank's
stage compute without the (< 0.1%) halo exchange.

    python tools/shard_modes.py            # prints one line per (cfg, N, mode)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import _lib, synth  # noqa: E402


def time_shard(dm, f, out, work, reps):
    for _ in range(2):
        dm.despeckle(f, out=out, work=work, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dm.despeckle(f, out=out, work=work, check=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    for key, total in (("c3", 256), ("c5", 32)):
        cfg = synth.CONFIGS[key]
        model = synth.config_model(cfg)
        base = np.stack([synth.noisy_image(cfg, i)[1] for i in range(4)])
        dm = tn.device_model_for(model)
        for n in (1, 2, 4, 8):
            B = total // n
            f = torch.from_numpy(base[np.arange(B) % 4]).cuda()
            out, work = torch.empty_like(f), torch.empty_like(f)
            reps = max(2, min(20, 64 // B))
            res = {}
            for mode in (0, 4, 6):
                _lib.set_stage_kernel(mode)
                res[mode] = time_shard(dm, f, out, work, reps)
            _lib.set_stage_kernel(0)
            px = B * cfg.H * cfg.W
            print(f"{key} N={n} B={B}: " + "  ".join(
                f"mode{m} {ms:.3f} ms {px / ms / 1e3:.1f} MPix/s" for m, ms in res.items()),
                flush=True)

    cfg = synth.CONFIGS["c4"]
    model = synth.config_model(cfg)
    dm = tn.device_model_for(model)
    tile = synth.noisy_image(cfg, 0, 1024, 1024)[1]
    base_ms = None
    for n in (1, 2, 4, 8):
        rows = cfg.H // n + (2 * (cfg.m - 1) if n > 1 else 0)
        f = torch.from_numpy(np.tile(tile, (rows // 1024 + 1, cfg.W // 1024))[:rows]).cuda()
        out, work = torch.empty_like(f), torch.empty_like(f)
        ms = time_shard(dm, f, out, work, 3)
        base_ms = base_ms or ms
        print(f"c4 N={n} strip {rows}x{cfg.W}: {ms:.3f} ms, scene-rate {cfg.H * cfg.W / (ms * 1e3):.1f} MPix/s "
              f"(ideal {base_ms / n:.3f} ms, efficiency {base_ms / n / ms:.3f})", flush=True)
        del f, out, work


if __name__ == "__main__":
    main()
