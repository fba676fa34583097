"""Row-strip sharding (C4's multi-GPU path) on CPU: world_size 2 and 3 gloo
process groups run the real partitioning + per-stage halo exchange with the
float64 oracle as the stage operator; the stitched strips must equal the
whole-image oracle (the halo makes each strip's interior exact)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1702_07482_b200 import strips, synth

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_strip_bounds_partition():
    for H in (1, 7, 61, 16384):
        for world in (1, 2, 3, 8):
            if world > H:
                continue
            b = [strips.strip_bounds(H, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == H
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(r1 - r0 for r0, r1 in b) - min(r1 - r0 for r0, r1 in b) <= 1


def test_strip_thinner_than_halo_rejected():
    lay = strips.StripLayout(10, 8, 4, 1, halo=6)
    with pytest.raises(ValueError, match="thinner"):
        lay.check()


@pytest.mark.parametrize("world,m", [(2, 7), (3, 5)])
def test_gloo_strips_match_whole_image_oracle(oracle, tmp_path, world, m):
    port = _free_port()
    H, W = 61, 45
    procs = []
    for r in range(world):
        procs.append(subprocess.Popen(
            [sys.executable, os.path.join(HERE, "helpers", "strip_worker.py"),
             "--rank", str(r), "--world", str(world), "--port", str(port),
             "--out", str(tmp_path / f"r{r}.npy"), "--H", str(H), "--W", str(W),
             "--m", str(m)]))
    for p in procs:
        assert p.wait(timeout=300) == 0
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)])
    model = synth.make_model(m, 5, 3, 63, seed=11)
    f = np.random.default_rng(3).uniform(0, 255, (H, W))
    ref = oracle.run_diffusion(f, model)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref) / ref) < 1e-12
