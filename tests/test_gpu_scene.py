"""Banded host path for one large scene (tnrd_plan_despeckle_host on a single
image of >= 2 x 3 waves of large tiles): row bands on their own streams
with event-ordered H2D / stages / D2H must give the BIT-identical result of
the whole-image device despeckle (band boundaries sit on the tile grid and
read their neighbours' rows in place), including the status contract."""
import numpy as np
import pytest

import paper_1702_07482_b200 as tn
from paper_1702_07482_b200 import synth

pytestmark = pytest.mark.gpu


def _scene(H, W):
    return np.ascontiguousarray(synth.scene_crop(synth.CONFIGS["c4"], 0, H, 0, W), dtype=np.float32)


@pytest.mark.parametrize("H,W", [(2048, 4096), (3072, 4096), (3000, 4100)])
def test_banded_host_bit_identical_to_whole_image(cuda, H, W):
    torch = __import__("torch")
    cfg = synth.CONFIGS["c2"]
    model = synth.config_model(cfg)
    dm = tn.device_model_for(model)
    f = _scene(H, W)
    whole = dm.despeckle(torch.from_numpy(f).cuda()).cpu().numpy()
    banded = dm.despeckle_host(f)
    assert np.array_equal(banded, whole)
    # repeated calls reuse the plan's band streams and events
    again = dm.despeckle_host(f)
    assert np.array_equal(again, whole)


def test_banded_host_status_contract(cuda):
    cfg = synth.CONFIGS["c2"]
    model = synth.config_model(cfg)
    dm = tn.device_model_for(model)
    f = np.full((3072, 4096), 100.0, dtype=np.float32)
    f[2900, 17] = -1.0        # in the last band
    with pytest.raises(ValueError):
        dm.despeckle_host(f)
    f[2900, 17] = np.inf
    with pytest.raises(ValueError):
        dm.despeckle_host(f)
    f[2900, 17] = 100.0
    u = dm.despeckle_host(f)   # the plan recovers after a failed call
    assert np.all(np.isfinite(u))
