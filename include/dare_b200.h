/*
 * dare_b200.h -- C ABI of the B200-native DARE hot paths (libdare_b200.so).
 *
 * Drop-in seam for the reference package `dare` (arxiv/paper_2605_26325,
 * pkg/src/dare/).  The reference is pure Python; its operator seam is the
 * numba kernels in _kernels.py plus the vectorised numpy blocks of
 * VolumeBuilder / compound / fill_holes.  Each entry point below names the
 * reference interface it replaces.  Plain pointers, sizes and opaque handles
 * only (no torch / C++ types); a ctypes binding is in INTEGRATION.md.
 *
 * Conventions
 *  - Every function returns 0 on success or a negative dare_status; the
 *    message is available from dare_last_error() (thread-local).
 *  - Preconditions that the reference checks in Python (unit-norm plane
 *    rotation, radius > 0, ...) are validated by the Python host layer before
 *    any call; these functions check only memory/shape consistency.
 *  - Host-computed f64 parameters are passed by value / host arrays so their
 *    bits are exactly what Python computed.
 *  - Re-entrant: concurrent calls on one (immutable) volume handle from many
 *    threads are safe; each calling thread gets its own CUDA stream.
 *  - `*_device` variants take device pointers and an explicit cudaStream_t
 *    (passed as void*) and do not synchronise; plain variants take host
 *    buffers, copy in/out and return when results are on the host.
 *
 * Plane parameters (14 doubles per pose, reslice.py:135-148 `_plane_params`):
 *   tx, ty, tz, r00, r01, r02, r10, r11, r12, r20, r21, r22, pitch_x, pitch_y
 * with R the (un-renormalised) plane rotation matrix, row-major.
 *
 * Frame axes (9 doubles per synchronized frame, reconstruct.py:152-163):
 *   R[0][0], R[1][0], R[2][0]   (image x axis  = R[:,0])
 *   R[0][1], R[1][1], R[2][1]   (image y axis  = R[:,1])
 *   tx, ty, tz                  (frame translation)
 */
#ifndef DARE_B200_H
#define DARE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DARE_OK = 0,
  DARE_ERR_INVALID = -1, /* bad argument / shape */
  DARE_ERR_CUDA = -2,    /* CUDA runtime error */
  DARE_ERR_NOMEM = -3,   /* device or host allocation failed */
  DARE_ERR_LIMIT = -4    /* input exceeds a documented layout limit */
} dare_status;

typedef struct dare_volume_s* dare_volume_t; /* sealed DirectionalVolume on one device */
typedef struct dare_scalar_s* dare_scalar_t; /* ScalarVolume on one device */

/* reslice.py:63-100 ResliceConfig, already reduced to kernel scalars
 * (cos_* = math.cos(math.radians(deg)) computed by the caller). */
typedef struct {
  double radius;
  double cos_normal;
  double cos_inplane;
  double k_normal;
  double k_inplane;
  double k_dist;
  int32_t unassigned;
  int32_t schedule; /* 0 auto, 1 pixel-major (spatially sorted batch), 2 pose-major
                       (lanes = one pixel of 32 consecutive poses; auto picks it for
                       coherent trajectories on the exact path only).  Results are
                       identical; only speed differs. */
  int32_t exact;    /* 0: certified f32 weights with exact-FP64 fallback for every
                       pixel whose u8 value / coverage the error bound cannot decide
                       (default); 1: FP64 reference arithmetic for every pixel.
                       Both produce the reference's pixels bit-for-bit. */
  int32_t _pad;
} dare_reslice_cfg;

typedef struct {
  int32_t device;
  int32_t _pad;
  double origin[3];
  double voxel_size;
  int64_t dims[3];
  int64_t n_samples;
  int64_t n_orientations;
  int64_t rejected_out_of_bounds;
  /* device pointers (read-only views, owned by the handle) */
  const uint32_t* d_cell_offsets; /* ncells + 1 exclusive prefix of counts */
  const void* d_records;          /* n_samples x 16 B: f32 x,y,z, u32 (oid<<8 | intensity),
                                     per cell grouped by z quarter (see d_bins / d_perm) */
  const float* d_orientations;    /* n_orientations x 4 f32 (w,x,y,z), canonical */
  const uint32_t* d_bins;         /* ncells: z-quarter bin bounds (b1 | b2<<8 | b3<<16 | 1<<24)
                                     of cells stored grouped by z quarter, 0 otherwise */
  const int8_t* d_perm;           /* n_samples: the cell's j-th sample in insertion order
                                     (index J = offsets[c] + j) is stored at J + perm[J] */
  size_t device_bytes;  /* all buffers of the handle, incl. the direction-cluster index of a
                           multi-direction volume once the first certified reslice built it */
} dare_volume_info;

typedef struct {
  int32_t device;
  int32_t _pad;
  double origin[3];
  double voxel_size;
  int64_t dims[3];
  float* d_values;   /* ncells f32 */
  uint8_t* d_flags;  /* ncells u8: 0 empty, 1 observed, 2 filled */
  int64_t* d_counts; /* ncells i64 observation counts, or NULL */
} dare_scalar_info;

/* ---- runtime ------------------------------------------------------------ */
const char* dare_last_error(void);
int dare_version(void);
int dare_get_device_count(int32_t* count);
int dare_set_device(int32_t device);
int dare_synchronize(void);
int dare_host_alloc(size_t bytes, void** ptr); /* pinned host memory */
int dare_host_free(void* ptr);
int dare_device_alloc(size_t bytes, void** ptr);
int dare_device_free(void* ptr);
int dare_memcpy(void* dst, const void* src, size_t bytes, void* stream); /* cudaMemcpyDefault */
int dare_stream_sync(void* stream);
/* Start-up for a process / service: makes `device` current, creates the
 * calling thread's stream and runs the one-time exhaustive check of the
 * hardware ex2/sqrt approximations that the certified reslice path relies on
 * (dare_fastmath_check), so the first reslice request does not pay it. */
int dare_init(int32_t device);
/* Returns unused memory of the current device's stream-ordered pool (volumes
 * and build scratch come from it; its release threshold is unlimited so that
 * rebuilds reuse memory) to the driver, keeping at most keep_bytes reserved.
 * Synchronises the device. */
int dare_trim(size_t keep_bytes);
/* Device span (ms, CUDA events on the call's stream, entry to completion) of
 * the last dare_reconstruct / dare_compound / dare_fill_holes call on this
 * thread; -1 before the first.  Lets a host measure kernel time without a
 * profiler. */
int dare_last_device_ms(double* ms);

/* ---- directional volume ------------------------------------------------- */

/* Replaces reconstruct.py:166-199 reconstruct_volume's per-frame scatter
 * (reconstruct.py:186-196, frame_world_positions 152-163, VolumeBuilder
 * insert_batch/_voxel_indices volume.py:208-238) and VolumeBuilder.seal
 * (volume.py:240-269).  `frames` is the (n_images, H, W) u8 stack (host or
 * device, see frames_on_device); frame_image[i] selects the image of the i-th
 * synchronized frame; axes/quats are per synchronized frame; mask (H*W u8,
 * host) or NULL.  Builds the sealed CSR volume on the current device and
 * reports the out-of-bounds count (volume.py:230-233). */
int dare_reconstruct(const uint8_t* frames, int64_t n_images, int32_t height, int32_t width,
                     int32_t frames_on_device, const int32_t* frame_image, int64_t n_frames,
                     const double* frame_axes, const float* frame_quats, double pitch_x,
                     double pitch_y, const uint8_t* mask, const double* origin, double voxel_size,
                     const int64_t* dims, dare_volume_t* out, int64_t* rejected_out_of_bounds);

/* Replaces VolumeBuilder.seal (volume.py:240-269) for arbitrary samples
 * (VolumeBuilder.insert_sample/insert_batch inputs, volume.py:211-238):
 * positions f32[n,3], orientations f32[n,4], intensities u8[n] in insertion
 * order (host).  Stable by insertion order within each cell, like numpy's
 * argsort(kind="stable"); out-of-bounds samples are dropped. */
int dare_volume_seal(const double* origin, double voxel_size, const int64_t* dims,
                     int64_t n_samples, const float* positions, const float* orientations,
                     const uint8_t* intensities, dare_volume_t* out);

/* Frame-sharded reconstruction (multi-GPU): merges n_parts partial
 * volumes built by dare_reconstruct over consecutive frame blocks into the
 * SAME grid.  Parts are device buffers on the current device (the d_* views
 * of dare_volume_info, or the same arrays received through NCCL): per part
 * the ncells+1 offsets, the 16 B records in the part's storage order with its
 * perm (insertion order is read through it; NULL perm array or entry = records
 * already in insertion order), the orientation table and its sizes.  Within
 * each cell the parts' runs are concatenated in part order -- the reference's
 * insertion order when part r holds frames after part r-1 -- and orientation
 * tables are deduplicated in part order, so the result (records, orientation
 * ids, bins, perm) is bit-identical to a single-device build. */
int dare_volume_merge(const double* origin, double voxel_size, const int64_t* dims,
                      int32_t n_parts, const uint32_t* const* d_offsets,
                      const void* const* d_records, const int8_t* const* d_perm,
                      const float* const* d_orient, const int64_t* n_samples,
                      const int64_t* n_orient, const int64_t* rejected, dare_volume_t* out);

/* Uploads a sealed volume in the reference layout (volume.py:76-93, as
 * produced by VolumeBuilder.seal or load_volume volume.py:300-330):
 * cell_starts/cell_counts i64[ncells], positions f32[n,3], orientations
 * f32[n,4], intensities u8[n] (host). */
int dare_volume_upload(const double* origin, double voxel_size, const int64_t* dims,
                       const int64_t* cell_starts, const int64_t* cell_counts, int64_t n_samples,
                       const float* positions, const float* orientations,
                       const uint8_t* intensities, dare_volume_t* out);

/* Materialises the reference layout on the host (buffers sized per info). */
int dare_volume_download(dare_volume_t vol, int64_t* cell_starts, int64_t* cell_counts,
                         float* positions, float* orientations, uint8_t* intensities);
/* Streaming .darevol writer (volume.py:272-297 save_volume): emits the exact
 * bytes of the reference file -- header, cell table, samples in insertion
 * order -- through `write(ctx, data, bytes)` (return 0 to continue) in chunks
 * of about chunk_bytes (0: 64 MB), double-buffered through pinned memory, so a
 * volume of any size is written with two chunks of host memory. */
typedef int (*dare_write_fn)(void* ctx, const void* data, size_t bytes);
int dare_volume_save_stream(dare_volume_t vol, dare_write_fn write, void* ctx, size_t chunk_bytes);
int dare_volume_get_info(dare_volume_t vol, dare_volume_info* info);
/* Frees the volume after synchronising its device (so reslices still queued
 * on caller streams by dare_reslice_device finish first). */
int dare_volume_destroy(dare_volume_t vol);

/* Replaces reslice.py:168-187 reslice -> _run_rows -> _kernels.reslice_rows_grid
 * (_kernels.py:84-139, _accumulate_run 29-68, _finalize_pixel 71-81), batched
 * over n_poses planes of one raster size.  params: n_poses x 14 doubles.
 * pixels/coverage: n_poses x height x width u8 (coverage 0/1).  Host buffers. */
int dare_reslice(dare_volume_t vol, int32_t n_poses, const double* params, int32_t width,
                 int32_t height, const dare_reslice_cfg* cfg, uint8_t* pixels,
                 uint8_t* coverage);
/* Host-side pose pipeline (no device work) for n synchronized frames, replacing
 * the per-frame Python of synchronize() after interpolation (reconstruct.py:119-149:
 * marker.compose(calibration) = normalised qmul + rotate(q, t_cal) + t,
 * geometry.py:69-77, 99-107, 128-133), the frame axes (rotation_matrix,
 * geometry.py:79-88; reconstruct.py:155-162), the canonical f32 quaternions
 * (reconstruct.py:192-195) and the image corners of compute_bounds
 * (volume.py:57-73).  mq n x 4 marker quaternions (w,x,y,z), mt n x 3; cal_q[4],
 * cal_t[3].  Outputs: rot n x 4, trans n x 3, axes n x 9 (R[:,0], R[:,1], t),
 * quats32 n x 4, lo[3] / hi[3] = compute_bounds' corner box before the
 * margin (sequential np.minimum / np.maximum).  *status: 0 ok, 1 zero quaternion (frame
 * *bad), 2 marker quaternion not unit (*bad, norm *bad_norm), 3 frame rotation
 * not unit (corners; *bad, *bad_norm) -- the caller raises the reference's error. */
int dare_frame_poses(int64_t n, const double* mq, const double* mt, const double* cal_q,
                     const double* cal_t, int32_t width, int32_t height, double px, double py,
                     double* rot, double* trans, double* axes, float* quats32, double* lo,
                     double* hi, int32_t* status, int64_t* bad, double* bad_norm);
/* Pose interpolation of synchronize() (reconstruct.py:102-116, slerp
 * geometry.py:159-180) for n frames at times t[j] strictly inside the pose
 * stream interval [ts[idx[j]], ts[idx[j]+1]] (idx = searchsorted(ts, t,
 * "right") - 1, computed by the caller): marker quaternions out_q n x 4 and
 * translations out_t n x 3, the reference's bits (host only, no device). */
int dare_interpolate_poses(int64_t n, const double* t, const int64_t* idx, const double* ts,
                           const double* pose_q, const double* pose_t, double* out_q, double* out_t);
/* Service form of dare_reslice (service.py:273-293 process_request, which
 * reslices one request and ships protocol.pack_coverage(image.coverage),
 * protocol.py:273-274): same pixels; coverage bit-packed on the device per pose
 * in np.packbits order (MSB first), ceil(height*width/8) bytes per pose, so the
 * device->host copy carries 1/8 of the coverage bytes.  Host buffers:
 * pixels n_poses x height x width, coverage_bits n_poses x ceil(h*w/8). */
int dare_reslice_packed(dare_volume_t vol, int32_t n_poses, const double* params, int32_t width,
                        int32_t height, const dare_reslice_cfg* cfg, uint8_t* pixels,
                        uint8_t* coverage_bits);
/* Contract twin of reslice (reslice.py:190-205 -> _kernels.reslice_rows_bruteforce
 * 142-167): every sample in storage order for every pixel.  Host buffers. */
int dare_reslice_bruteforce(dare_volume_t vol, int32_t n_poses, const double* params,
                            int32_t width, int32_t height, const dare_reslice_cfg* cfg,
                            uint8_t* pixels, uint8_t* coverage);
/* Same on device buffers (params, pixels, coverage device pointers). */
int dare_reslice_device(dare_volume_t vol, int32_t n_poses, const double* d_params,
                        int32_t width, int32_t height, const dare_reslice_cfg* cfg,
                        uint8_t* d_pixels, uint8_t* d_coverage, void* stream);

/* 1 when consecutive planes of the batch are close (centre within one voxel,
 * rotation within ~3 degrees) for >= 90% of pairs and n_poses >= 32: the
 * pose-major schedule then shares every load across the warp.  Host params. */
int dare_poses_coherent(const double* params, int32_t n_poses, int32_t width, int32_t height,
                        double voxel_size);

/* ---- scalar (direction-blind) arm -------------------------------------- */

/* Replaces baseline.py:64-97 compound (np.add.at scatter + mean). Arguments
 * as dare_reconstruct. */
int dare_compound(const uint8_t* frames, int64_t n_images, int32_t height, int32_t width,
                  int32_t frames_on_device, const int32_t* frame_image, int64_t n_frames,
                  const double* frame_axes, double pitch_x, double pitch_y, const uint8_t* mask,
                  const double* origin, double voxel_size, const int64_t* dims,
                  dare_scalar_t* out);
/* The two halves of dare_compound, for frame-sharded compounding: accumulate
 * the frames' u64 intensity sums and observation counts into caller-owned,
 * zero-initialised device arrays (ncells each; exact integers, so per-rank
 * partials combine with an all-reduce SUM), then finalise values/flags. */
int dare_compound_accumulate(const uint8_t* frames, int64_t n_images, int32_t height,
                             int32_t width, int32_t frames_on_device, const int32_t* frame_image,
                             int64_t n_frames, const double* frame_axes, double pitch_x,
                             double pitch_y, const uint8_t* mask, const double* origin,
                             double voxel_size, const int64_t* dims, uint64_t* d_sums,
                             uint64_t* d_counts, void* stream);
int dare_scalar_from_sums(const double* origin, double voxel_size, const int64_t* dims,
                          const uint64_t* d_sums, const uint64_t* d_counts, dare_scalar_t* out);
/* Creates a scalar volume from values f32 / flags u8 / counts i64 (counts may
 * be NULL), host or device pointers (unified addressing: e.g. buffers received
 * through an NCCL broadcast are copied device-to-device). */
int dare_scalar_upload(const double* origin, double voxel_size, const int64_t* dims,
                       const float* values, const uint8_t* flags, const int64_t* counts,
                       dare_scalar_t* out);
int dare_scalar_download(dare_scalar_t vol, float* values, uint8_t* flags, int64_t* counts);
int dare_scalar_get_info(dare_scalar_t vol, dare_scalar_info* info);
int dare_scalar_destroy(dare_scalar_t vol);

/* Replaces baseline.py:100-127 fill_holes (Jacobi passes, bit-exact). Returns
 * a new handle; *passes_run = passes that filled at least one voxel. */
int dare_fill_holes(dare_scalar_t in, int32_t max_passes, dare_scalar_t* out,
                    int32_t* passes_run);

/* Replaces baseline.py:130-155 reslice_trilinear -> _kernels.trilinear_rows
 * (_kernels.py:170-229), batched.  values (optional, may be NULL) receives the
 * pre-rounding f64 value per pixel.  Host buffers. */
int dare_reslice_trilinear(dare_scalar_t vol, int32_t n_poses, const double* params,
                           int32_t width, int32_t height, uint8_t* pixels, uint8_t* coverage,
                           double* values);
int dare_reslice_trilinear_device(dare_scalar_t vol, int32_t n_poses, const double* d_params,
                                  int32_t width, int32_t height, uint8_t* d_pixels,
                                  uint8_t* d_coverage, double* d_values, void* stream);

/* ---- evaluation --------------------------------------- */
enum { DARE_ELEM_U8 = 0, DARE_ELEM_F64 = 1 };
/* Replaces evaluation.py:41-84 ncc / ssim (uniform window, unbiased
 * covariance, complete windows only) and compare_images (evaluation.py:150-160)
 * for n_pairs image pairs a[p], b[p] of height x width (element type
 * DARE_ELEM_U8 or DARE_ELEM_F64, [n_pairs][height][width]); a_mask / b_mask u8
 * of the same shape or NULL (all valid).  Per pair: ncc, ssim, valid (mask
 * intersection count) and status bits: 1 fewer than 2 valid pixels, 2 zero
 * variance (ncc undefined), 4 no complete window, 8 image smaller than the
 * window (ssim undefined).  SSIM is bit-identical to the reference for
 * integer-valued images (the NCC dot products agree to rounding).  window odd
 * and >= 3.  Host buffers; _device: device buffers on `stream`. */
int dare_similarity(int32_t n_pairs, int32_t height, int32_t width, int32_t elem, const void* a,
                    const uint8_t* a_mask, const void* b, const uint8_t* b_mask, int32_t window,
                    double c1, double c2, double* ncc, double* ssim, int64_t* valid,
                    int32_t* status);
int dare_similarity_device(int32_t n_pairs, int32_t height, int32_t width, int32_t elem,
                           const void* d_a, const uint8_t* d_a_mask, const void* d_b,
                           const uint8_t* d_b_mask, int32_t window, double c1, double c2,
                           double* d_ncc, double* d_ssim, int64_t* d_valid, int32_t* d_status,
                           void* stream);

/* ---- diagnostics -------------------------------------------------------- */
/* Device restatement of glibc exp on n device doubles (parity tests). */
int dare_exp_device(const double* d_x, double* d_y, int64_t n, void* stream);
/* Host-only diagnostic: the exact per-axis threshold tables the count and
 * compound passes use for a grid (T[k] = smallest f64 world coordinate whose
 * reference cell index floor((f64(f32(P)) - o) / v) is >= k; with zfine the z
 * table interleaves the z-quarter bin bounds).  out holds (nx+1) + (ny+1) +
 * (nz+1, or 4 nz + 1 with zfine) doubles; n_out[3] = intervals per table
 * (-1 when the fine table is not monotone). */
int dare_cell_thresholds(const double* origin, double voxel_size, const int64_t* dims, int32_t zfine,
                         double* out, int64_t* n_out);
/* Pixels the last dare_reslice / dare_reslice_bruteforce call on this thread
 * recomputed on the exact FP64 path because the certified bound was
 * inconclusive (0 with cfg.exact = 1, or when the fast path is disabled). */
int dare_reslice_last_fallback(int64_t* n_pixels);
/* Exhaustive check (every f32 input of the ranges the certified reslice path
 * uses) of the hardware ex2.approx / sqrt.approx relative error on the
 * current device; *ok = 1 when both are within the constants the bound
 * assumes.  The fast path runs this once per device and disables itself
 * (exact FP64 for every pixel) if it fails. */
int dare_fastmath_check(double* ex2_max_rel_err, double* sqrt_max_rel_err, int32_t* ok);

#ifdef __cplusplus
}
#endif
#endif /* DARE_B200_H */
