"""B200-native (sm_100a) 3D Surface Splatting hot path.

Drop-in for the reference package's render / backward_image / loss /
Adam.step / refine_topology path (surfsplat 0.1.0).  Every entry point runs
hand-written CUDA kernels from csrc/ through the C ABI in include/ss_abi.h;
there is no CPU fallback.
"""

from .camera import Camera, fibonacci_cameras, look_at, orbit_cameras, perspective_matrix
from .surfels import SurfelCloud, logit, quats_from_normals
from .preprocess import PreprocessOptions, ProjectedSurfels, preprocess
from .rasterizer import RenderOptions, RenderResult, bin_and_sort, render
from .backward import BackwardResult, backward_image
from .shading import EnvironmentLight, brdf_lut, shade_surfels, tone_map, tone_map_backward
from .losses import image_loss, normal_consistency_loss, photometric_loss, silhouette_loss, ssim_loss
from .knn import NeighborIndex
from .adam import Adam, normalize_quats
from .densify import DensifyStats, mask_votes, prune_keep_mask, refine_topology, select_split, split_cloud
from .step import TrainStep
from . import sceneio

__version__ = "0.1.0"

__all__ = ["Camera", "fibonacci_cameras", "look_at", "orbit_cameras", "perspective_matrix", "SurfelCloud",
           "logit", "quats_from_normals", "PreprocessOptions", "ProjectedSurfels", "preprocess", "RenderOptions",
           "RenderResult", "bin_and_sort", "render", "BackwardResult", "backward_image", "EnvironmentLight",
           "brdf_lut", "shade_surfels", "tone_map", "tone_map_backward", "photometric_loss", "silhouette_loss",
           "ssim_loss", "image_loss", "normal_consistency_loss", "NeighborIndex",
           "Adam", "normalize_quats", "DensifyStats", "mask_votes", "prune_keep_mask", "refine_topology",
           "select_split", "split_cloud", "TrainStep", "sceneio"]
