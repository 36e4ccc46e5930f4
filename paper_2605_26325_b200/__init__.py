"""B200-native DARE hot paths: directional reconstruction, normalisation /
gap filling, and direction-aware reslicing as hand-written sm_100a CUDA
kernels behind a C ABI (include/dare_b200.h), with a Python host layer that
mirrors the reference package `dare` (arxiv/paper_2605_26325, pkg/src/dare).

Drop-in surface (same names, signatures, defaults, errors as the reference):
  reconstruct_volume, reslice, reslice_bruteforce, compound, fill_holes,
  reslice_trilinear, trilinear_at_points, VolumeBuilder, DirectionalVolume,
  ScalarVolume, ReslicePlane, ResliceConfig, ResliceImage, SweepRecording,
  save/load_volume, save/load_scalar_volume, geometry types.
B200 extensions: reslice_batch, reslice_trilinear_batch (many poses per
launch), reconstruct_volume(frames_device_ptr=...), parallel.* (multi-GPU),
service.ResliceBatcher / reslice_packed (service request path: concurrent
requests coalesced into batched launches, coverage bit-packed on device).
"""
from .errors import (
    DareError,
    InvalidArgumentError,
    OutOfBoundsError,
    ProtocolError,
    SweepFormatError,
    SynchronizationError,
    UndefinedMetricError,
    VolumeFormatError,
)
from .geometry import FrameAxes, Pose, Quaternion, frame_axes, rotate, slerp
from .sweep import SweepRecording, TrackedFrame, interpolate_pose, pixel_to_world, synchronize
from .volume import (
    BoundingBox,
    DirectionalSample,
    DirectionalVolume,
    VolumeBuilder,
    as_device_volume,
    compute_bounds,
    load_volume,
    save_volume,
)
from .reslice import (
    ReslicePlane,
    ResliceConfig,
    ResliceImage,
    accept,
    directional_dots,
    reslice,
    reslice_batch,
    reslice_bruteforce,
    sample_weight,
)
from .reconstruct import reconstruct_volume
from .service import ResliceBatcher, reslice_packed
from .scalar import (
    VOXEL_EMPTY,
    VOXEL_FILLED,
    VOXEL_OBSERVED,
    ScalarVolume,
    compound,
    fill_holes,
    load_scalar_volume,
    reslice_trilinear,
    reslice_trilinear_batch,
    save_scalar_volume,
    trilinear_at_points,
)

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
