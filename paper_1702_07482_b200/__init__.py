"""B200-native TNRD despeckling inference (arXiv 1702.07482).

Drop-in for the inference path of the reference package ``specklediff``:
the same model containers and function names, with each diffusion stage
executed as one fused sm_100a CUDA kernel through a C ABI
(include/tnrd.h, libtnrd.so).  No CPU fallback.
"""
from .diffusion import (VARIANTS, DiffusionModel, StageParams, StageTrace,
                        default_rbf_grid, diffusion_force, diffusion_step,
                        diffusion_step_projected, initial_state,
                        projection_reaction, run_diffusion, run_diffusion_batch,
                        smooth_max, zero_mean_basis)
from .engine import DeviceModel, device_model_for
from .imageops import (as_image, as_kernel, conv2d, conv2d_adjoint, patch_correlation,
                       rotate180)
from .influence import RbfGrid
from .speckle import (F_FLOOR, NoisyPair, SpeckleConfig, prox_idiv,
                      nakagami_mean, sample_speckle, sample_speckle_device,
                      sample_speckle_gpu,
                      speckle_field, speckle_field_device)

__all__ = [
    "VARIANTS", "DiffusionModel", "StageParams", "StageTrace",
    "default_rbf_grid", "diffusion_force", "diffusion_step",
    "diffusion_step_projected", "initial_state", "run_diffusion",
    "run_diffusion_batch", "zero_mean_basis", "smooth_max", "projection_reaction",
    "DeviceModel",
    "device_model_for", "as_image", "as_kernel", "conv2d", "rotate180",
    "conv2d_adjoint", "patch_correlation",
    "RbfGrid", "F_FLOOR", "NoisyPair", "SpeckleConfig", "prox_idiv",
    "sample_speckle", "speckle_field", "sample_speckle_device",
    "sample_speckle_gpu", "speckle_field_device", "nakagami_mean",
]

__version__ = "0.1.0"
