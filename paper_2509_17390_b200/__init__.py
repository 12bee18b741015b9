"""B200-native LiDAR first-return ray casting (the hot path of FGGS-LiDAR, arXiv 2509.17390 §IV-C).

The compute lives in libfgl.so (csrc/, sm_100a); `fgl` is its ctypes binding and `dist` the
multi-GPU pose sweep over torch.distributed. See DESIGN.md.
"""
from .fgl import (FglError, GaussianScene, denoise, denoise_quantile, marching_cubes, tsdf, PointCloud, Scene, cloud_metrics, export_rays, kernel_launches, l2_read_probe, lib, morton_codes, rays_per_pose, sort_pairs,  # noqa: F401
                  version, LIB_PATH, SYMBOLS)

__all__ = ["FglError", "GaussianScene", "denoise", "denoise_quantile", "marching_cubes", "tsdf", "PointCloud", "Scene", "cloud_metrics", "export_rays", "kernel_launches", "l2_read_probe", "lib", "morton_codes", "rays_per_pose", "sort_pairs", "version",
           "LIB_PATH", "SYMBOLS"]
