"""Probe: does splitting a batch shard into sub-batches on k streams fill the
tail wave of each stage?  Images are independent, so stage t + 1 of one
sub-batch can run while stage t of another drains.  Times one shard of
C3 / C5 (the per-rank shards of bench.py --gpus N) single-stream vs k
streams; outputs are checked bit-identical.

    python tools/multistream_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_07482_b200 as tn  # noqa: E402
from paper_1702_07482_b200 import synth  # noqa: E402


def run(dm, f, out, work, streams):
    k = len(streams)
    B = f.shape[0]
    cuts = [B * i // k for i in range(k + 1)]
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for s, a, b in zip(streams, cuts[:-1], cuts[1:]):
        if b > a:
            dm.despeckle(f[a:b], out=out[a:b], work=work[a:b], stream=s, check=False)
    for s in streams:
        cur.wait_stream(s)


def timed(dm, f, out, work, streams, reps):
    for _ in range(2):
        run(dm, f, out, work, streams)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run(dm, f, out, work, streams)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    for key, Bs in (("c3", (256, 32, 64)), ("c5", (32, 4, 8))):
        cfg = synth.CONFIGS[key]
        model = synth.config_model(cfg)
        base = np.stack([synth.noisy_image(cfg, i)[1] for i in range(4)])
        dm = tn.device_model_for(model)
        for B in Bs:
            f = torch.from_numpy(base[np.arange(B) % 4]).cuda()
            out, work = torch.empty_like(f), torch.empty_like(f)
            reps = max(2, min(20, 64 // B))
            ref = None
            line = []
            for k in (1, 2, 4):
                if k > B:
                    continue
                streams = [torch.cuda.Stream() for _ in range(k)]
                ms = timed(dm, f, out, work, streams, reps)
                if ref is None:
                    ref = out.clone()
                same = bool(torch.equal(out, ref))
                px = B * cfg.H * cfg.W
                line.append(f"k={k} {ms:.3f} ms {px / ms / 1e3:.1f} MPix/s{'' if same else ' MISMATCH'}")
            print(f"{key} B={B}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    main()
