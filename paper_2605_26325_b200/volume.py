"""Directional volume: device-resident CSR with lazily materialised host views.

Drop-in for pkg/src/dare/volume.py:1-330.  A DirectionalVolume here owns a
libdare_b200 handle (records/offsets in HBM, see csrc/volume.cuh); the
reference's host arrays (cell_starts, cell_counts, positions, orientations,
intensities) are produced on first access by one device->host download and
are read-only, exactly like the sealed reference volume.  A volume can also
be created from host arrays (the reference constructor signature, or a
reference DirectionalVolume via `as_device_volume`), in which case it is
uploaded on first device use.
"""
from __future__ import annotations

import ctypes
import struct
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidArgumentError, OutOfBoundsError, VolumeFormatError
from .geometry import Quaternion

VOLUME_MAGIC = b"DARE"
VOLUME_VERSION = 1
DEFAULT_VOXEL_SIZE_MM = 0.125
_HEADER = struct.Struct("<4sI3dd3IQ")  # volume.py:23
_TABLE = np.dtype([("offset", "<u8"), ("count", "<u4")])
_SAMPLE = np.dtype([("position", "<f4", 3), ("orientation", "<f4", 4), ("intensity", "u1"),
                    ("pad", "u1", 3)])


@dataclass(frozen=True)
class DirectionalSample:
    intensity: int
    orientation: Quaternion
    position: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "position", np.asarray(self.position, dtype=np.float32).reshape(3))


@dataclass(frozen=True)
class BoundingBox:
    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "min", np.asarray(self.min, dtype=float).reshape(3))
        object.__setattr__(self, "max", np.asarray(self.max, dtype=float).reshape(3))
        if np.any(self.min > self.max):
            raise InvalidArgumentError("bounding box min must be <= max componentwise")

    def expanded(self, margin: float) -> "BoundingBox":
        return BoundingBox(self.min - margin, self.max + margin)

    @property
    def extent(self) -> np.ndarray:
        return self.max - self.min


def compute_bounds(frames, margin: float = 0.0) -> BoundingBox:
    """Box over the four image corners of every frame (volume.py:57-73)."""
    from . import geometry as geo

    frames = list(frames)
    if not frames:
        raise InvalidArgumentError("compute_bounds requires at least one frame")
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    for f in frames:
        px, py = f.pixel_pitch
        umax = (f.width - 1) * px
        vmax = (f.height - 1) * py
        for u, v in ((0.0, 0.0), (umax, 0.0), (0.0, vmax), (umax, vmax)):
            c = geo.rotate(f.pose.rotation, (u, v, 0.0)) + f.pose.translation
            lo = np.minimum(lo, c)
            hi = np.maximum(hi, c)
    return BoundingBox(lo, hi).expanded(margin)


class _Handle:
    """Owns a dare_volume_t; destroyed with the Python object."""

    def __init__(self, raw: int):
        self.raw = ctypes.c_void_p(raw)
        self._fin = weakref.finalize(self, _destroy, raw)

    def info(self) -> _lib.VolumeInfo:
        info = _lib.VolumeInfo()
        _lib.call("dare_volume_get_info", self.raw, ctypes.byref(info))
        return info


def _destroy(raw: int) -> None:
    try:
        _lib.load().dare_volume_destroy(ctypes.c_void_p(raw))
    except Exception:
        pass


class DirectionalVolume:
    """Sealed, immutable directional volume (volume.py:76-186)."""

    def __init__(self, origin, voxel_size, dims, cell_starts=None, cell_counts=None,
                 positions=None, orientations=None, intensities=None, *, _handle: _Handle | None = None):
        self.origin = np.asarray(origin, dtype=float).reshape(3).copy()
        self.origin.flags.writeable = False
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(d) for d in dims)
        self._handle = _handle
        self._host = None
        self._lock = threading.Lock()
        self.rejected_out_of_bounds = 0
        if _handle is None:
            arrays = (cell_starts, cell_counts, positions, orientations, intensities)
            if any(a is None for a in arrays):
                raise InvalidArgumentError("host arrays required when no device handle is given")
            self._set_host(*arrays)
        else:
            info = _handle.info()
            self._n = int(info.n_samples)
            self.rejected_out_of_bounds = int(info.rejected_out_of_bounds)

    # ---- host views ------------------------------------------------------
    def _set_host(self, starts, counts, pos, quat, inten):
        arrs = (
            np.ascontiguousarray(starts, dtype=np.int64),
            np.ascontiguousarray(counts, dtype=np.int64),
            np.ascontiguousarray(pos, dtype=np.float32).reshape(-1, 3),
            np.ascontiguousarray(quat, dtype=np.float32).reshape(-1, 4),
            np.ascontiguousarray(inten, dtype=np.uint8).reshape(-1),
        )
        for a in arrs:
            a.flags.writeable = False
        self._host = arrs
        self._n = int(arrs[4].shape[0])

    def _host_arrays(self):
        if self._host is None:
            with self._lock:
                if self._host is None:
                    nc, n = self.cell_count, self._n
                    starts = np.empty(nc, np.int64)
                    counts = np.empty(nc, np.int64)
                    pos = np.empty((n, 3), np.float32)
                    quat = np.empty((n, 4), np.float32)
                    inten = np.empty(n, np.uint8)
                    _lib.call("dare_volume_download", self._handle.raw, _lib.ptr(starts, ctypes.c_int64),
                              _lib.ptr(counts, ctypes.c_int64), _lib.ptr(pos, ctypes.c_float),
                              _lib.ptr(quat, ctypes.c_float), _lib.ptr(inten, ctypes.c_uint8))
                    self._set_host(starts, counts, pos, quat, inten)
        return self._host

    @property
    def cell_starts(self) -> np.ndarray:
        return self._host_arrays()[0]

    @property
    def cell_counts(self) -> np.ndarray:
        return self._host_arrays()[1]

    @property
    def positions(self) -> np.ndarray:
        return self._host_arrays()[2]

    @property
    def orientations(self) -> np.ndarray:
        return self._host_arrays()[3]

    @property
    def intensities(self) -> np.ndarray:
        return self._host_arrays()[4]

    # ---- device handle -----------------------------------------------------
    def device_handle(self) -> _Handle:
        if self._handle is None:
            with self._lock:
                if self._handle is None:
                    self._handle = _upload(self.origin, self.voxel_size, self.dims, *self._host)
        return self._handle

    def device_info(self) -> _lib.VolumeInfo:
        return self.device_handle().info()

    # ---- reference API -----------------------------------------------------
    @property
    def sample_count(self) -> int:
        return self._n

    @property
    def cell_count(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    def linear_index(self, idx) -> int:
        ix, iy, iz = idx
        _, ny, nz = self.dims
        return (ix * ny + iy) * nz + iz

    def voxel_of(self, p):
        p = np.asarray(p, dtype=float)
        idx = np.floor((p - self.origin) / self.voxel_size).astype(np.int64)
        if np.any(idx < 0) or np.any(idx >= np.asarray(self.dims)):
            return None
        return (int(idx[0]), int(idx[1]), int(idx[2]))

    def cell_slice(self, idx) -> slice:
        lin = self.linear_index(idx)
        start = int(self.cell_starts[lin])
        return slice(start, start + int(self.cell_counts[lin]))

    def cell_range_for_cube(self, p, radius: float):
        p = np.asarray(p, dtype=float)
        lo = np.floor((p - radius - self.origin) / self.voxel_size - 1e-9).astype(np.int64)
        hi = np.floor((p + radius - self.origin) / self.voxel_size + 1e-9).astype(np.int64)
        lo = np.maximum(lo, 0)
        hi = np.minimum(hi, np.asarray(self.dims, dtype=np.int64) - 1)
        if np.any(lo > hi):
            return None
        return lo, hi

    def gather_indices(self, p, radius: float) -> np.ndarray:
        if radius <= 0:
            raise InvalidArgumentError("gather radius must be > 0")
        rng = self.cell_range_for_cube(p, radius)
        if rng is None:
            return np.empty(0, dtype=np.int64)
        lo, hi = rng
        _, ny, nz = self.dims
        starts, counts = self.cell_starts, self.cell_counts
        chunks = []
        for ix in range(lo[0], hi[0] + 1):
            for iy in range(lo[1], hi[1] + 1):
                base = (ix * ny + iy) * nz
                for lin in range(base + lo[2], base + hi[2] + 1):
                    if counts[lin]:
                        chunks.append(np.arange(starts[lin], starts[lin] + counts[lin], dtype=np.int64))
        return np.concatenate(chunks) if chunks else np.empty(0, dtype=np.int64)

    def sample_at(self, i: int) -> DirectionalSample:
        return DirectionalSample(int(self.intensities[i]),
                                 Quaternion(*(float(c) for c in self.orientations[i])),
                                 self.positions[i].copy())

    def gather_neighborhood(self, p, radius: float) -> list[DirectionalSample]:
        return [self.sample_at(i) for i in self.gather_indices(p, radius)]


def _upload(origin, voxel, dims, starts, counts, pos, quat, inten) -> _Handle:
    raw = ctypes.c_void_p()
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(dims, dtype=np.int64)
    _lib.call("dare_volume_upload", _lib.ptr(o, ctypes.c_double), float(voxel), _lib.ptr(d, ctypes.c_int64),
              _lib.ptr(starts, ctypes.c_int64), _lib.ptr(counts, ctypes.c_int64), int(len(inten)),
              _lib.ptr(pos, ctypes.c_float), _lib.ptr(quat, ctypes.c_float), _lib.ptr(inten, ctypes.c_uint8),
              ctypes.byref(raw))
    return _Handle(raw.value)


_foreign_cache: "weakref.WeakKeyDictionary[object, DirectionalVolume]" = weakref.WeakKeyDictionary()
_foreign_lock = threading.Lock()


def as_device_volume(volume) -> DirectionalVolume:
    """Accepts this package's volume or any object with the reference's
    DirectionalVolume attributes (e.g. a dare.volume.DirectionalVolume built
    by the reference); foreign volumes are uploaded once and cached (they are
    immutable, volume.py:89-92)."""
    if isinstance(volume, DirectionalVolume):
        return volume

    def convert():
        v = DirectionalVolume(volume.origin, volume.voxel_size, volume.dims, volume.cell_starts,
                              volume.cell_counts, volume.positions, volume.orientations, volume.intensities)
        v.rejected_out_of_bounds = getattr(volume, "rejected_out_of_bounds", 0)
        return v

    with _foreign_lock:
        try:
            cached = _foreign_cache.get(volume)
        except TypeError:  # not weak-referenceable: no caching
            return convert()
        if cached is None:
            cached = convert()
            _foreign_cache[volume] = cached
    return cached


class VolumeBuilder:
    """Accumulate samples, then seal on the device (volume.py:189-269)."""

    def __init__(self, bounds: BoundingBox, voxel_size: float = DEFAULT_VOXEL_SIZE_MM):
        if voxel_size <= 0:
            raise InvalidArgumentError("voxel_size must be > 0")
        self.origin = bounds.min.copy()
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(np.floor(e / voxel_size)) + 1 for e in bounds.extent)
        self._pos: list[np.ndarray] = []
        self._quat: list[np.ndarray] = []
        self._inten: list[np.ndarray] = []
        self.rejected_out_of_bounds = 0

    def _cells(self, pos32: np.ndarray) -> np.ndarray:
        return np.floor((pos32.astype(np.float64) - self.origin) / self.voxel_size).astype(np.int64)

    def insert_sample(self, s: DirectionalSample) -> None:
        pos = np.asarray(s.position, dtype=np.float32).reshape(1, 3)
        idx = self._cells(pos)[0]
        if np.any(idx < 0) or np.any(idx >= np.asarray(self.dims)):
            raise OutOfBoundsError(f"sample position {pos[0]} outside volume grid")
        q = s.orientation.normalized().canonical()
        self._pos.append(pos)
        self._quat.append(np.array([[q.w, q.x, q.y, q.z]], dtype=np.float32))
        self._inten.append(np.array([s.intensity], dtype=np.uint8))

    def insert_batch(self, positions, orientations, intensities) -> int:
        pos = np.ascontiguousarray(positions, dtype=np.float32).reshape(-1, 3)
        quat = np.ascontiguousarray(orientations, dtype=np.float32).reshape(-1, 4)
        inten = np.ascontiguousarray(intensities, dtype=np.uint8).reshape(-1)
        idx = self._cells(pos)
        ok = np.all((idx >= 0) & (idx < np.asarray(self.dims)), axis=1)
        n_bad = int(np.count_nonzero(~ok))
        self.rejected_out_of_bounds += n_bad
        if n_bad:
            pos, quat, inten = pos[ok], quat[ok], inten[ok]
        self._pos.append(pos)
        self._quat.append(quat)
        self._inten.append(inten)
        return n_bad

    def seal(self) -> DirectionalVolume:
        pos = np.ascontiguousarray(np.concatenate(self._pos) if self._pos else np.empty((0, 3), np.float32))
        quat = np.ascontiguousarray(np.concatenate(self._quat) if self._quat else np.empty((0, 4), np.float32))
        inten = np.ascontiguousarray(np.concatenate(self._inten) if self._inten else np.empty(0, np.uint8))
        raw = ctypes.c_void_p()
        o = np.ascontiguousarray(self.origin, dtype=np.float64)
        d = np.ascontiguousarray(self.dims, dtype=np.int64)
        _lib.call("dare_volume_seal", _lib.ptr(o, ctypes.c_double), self.voxel_size,
                  _lib.ptr(d, ctypes.c_int64), int(len(inten)), _lib.ptr(pos, ctypes.c_float),
                  _lib.ptr(quat, ctypes.c_float), _lib.ptr(inten, ctypes.c_uint8), ctypes.byref(raw))
        return DirectionalVolume(self.origin, self.voxel_size, self.dims, _handle=_Handle(raw.value))


def save_volume(volume, path, chunk_bytes: int = 64 << 20) -> None:
    """.darevol writer, byte-identical to volume.py:272-297.

    `path` is a file name or a writable binary file object.  A device volume
    whose host arrays were never materialised is streamed straight from HBM
    (dare_volume_save_stream: records read through perm in insertion order,
    chunks double-buffered through pinned memory), so saving a multi-GB volume
    needs two chunks of host memory, not the reference's full structured copy.
    """
    if isinstance(volume, DirectionalVolume) and volume._host is None and volume._handle is not None:
        def stream(fh):
            err = []

            def write(_ctx, data, nbytes):
                try:
                    fh.write(memoryview((ctypes.c_ubyte * nbytes).from_address(data)))
                    return 0
                except BaseException as e:  # noqa: BLE001 (re-raised below)
                    err.append(e)
                    return 1

            cb = _lib.WRITE_FN(write)
            try:
                _lib.call("dare_volume_save_stream", volume._handle.raw, cb, None, int(chunk_bytes))
            except Exception:
                if err:
                    raise err[0]
                raise

        if hasattr(path, "write"):
            stream(path)
        else:
            with open(path, "wb") as fh:
                stream(fh)
        return
    nc = int(np.prod(volume.dims))
    n = int(volume.intensities.shape[0])
    header = _HEADER.pack(VOLUME_MAGIC, VOLUME_VERSION, *[float(c) for c in volume.origin],
                          float(volume.voxel_size), *volume.dims, n)
    table = np.zeros(nc, dtype=_TABLE)
    table["offset"] = volume.cell_starts
    table["count"] = volume.cell_counts
    samples = np.zeros(n, dtype=_SAMPLE)
    samples["position"] = volume.positions
    samples["orientation"] = volume.orientations
    samples["intensity"] = volume.intensities

    def emit(fh):
        fh.write(header)
        fh.write(table.tobytes())
        fh.write(samples.tobytes())

    if hasattr(path, "write"):
        emit(path)
    else:
        with open(path, "wb") as fh:
            emit(fh)


def load_volume(path) -> DirectionalVolume:
    """.darevol reader (volume.py:300-330); uploads on first device use."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER.size:
        raise VolumeFormatError(f"{path}: truncated header")
    magic, version, ox, oy, oz, voxel, nx, ny, nz, count = _HEADER.unpack_from(raw, 0)
    if magic != VOLUME_MAGIC:
        raise VolumeFormatError(f"{path}: bad magic {magic!r}, expected {VOLUME_MAGIC!r}")
    if version != VOLUME_VERSION:
        raise VolumeFormatError(f"{path}: unsupported format version {version}")
    nc = nx * ny * nz
    off = _HEADER.size
    expected = off + nc * _TABLE.itemsize + count * _SAMPLE.itemsize
    if len(raw) != expected:
        raise VolumeFormatError(f"{path}: size {len(raw)} != expected {expected}")
    table = np.frombuffer(raw, dtype=_TABLE, count=nc, offset=off)
    samples = np.frombuffer(raw, dtype=_SAMPLE, count=count, offset=off + nc * _TABLE.itemsize)
    return DirectionalVolume((ox, oy, oz), voxel, (nx, ny, nz), table["offset"].astype(np.int64),
                             table["count"].astype(np.int64), np.ascontiguousarray(samples["position"]),
                             np.ascontiguousarray(samples["orientation"]),
                             np.ascontiguousarray(samples["intensity"]))
