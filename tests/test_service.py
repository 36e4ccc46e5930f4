"""Service request path (reference service.py:144-159,
273-334 and tests/test_service.py): validation + clamping on CPU, and on the
GPU the batched, device-packed path against the library's single reslices."""
import math
import threading

import numpy as np
import pytest

import paper_2605_26325_b200 as db
from oracle import oracle
from paper_2605_26325_b200 import service as svc
from paper_2605_26325_b200.geometry import Pose, Quaternion
from paper_2605_26325_b200.reslice import ReslicePlane, ResliceConfig


def _req(i, pose=(1.0, 2.0, 3.0, 1.0, 0.0, 0.0, 0.0), w=24, h=17, pitch=(0.2, 0.2), enc=0, config=None):
    return svc.ResliceRequest(i, tuple(pose), w, h, tuple(pitch), enc, config)


# ---- CPU: validation and clamping (service.py:295-334) --------------------------------------

def test_validate_request_messages():
    base = ResliceConfig()
    with pytest.raises(ValueError, match="not a unit quaternion"):
        svc.validate_request(_req(1, (0, 0, 0, 2.0, 0, 0, 0)), base, 0.25)
    with pytest.raises(ValueError, match="non-finite"):
        svc.validate_request(_req(1, (math.nan, 0, 0, 1.0, 0, 0, 0)), base, 0.25)
    with pytest.raises(ValueError, match="width/height must be 1..4096"):
        svc.validate_request(_req(1, w=0), base, 0.25)
    with pytest.raises(ValueError, match="width/height must be 1..4096"):
        svc.validate_request(_req(1, h=4097), base, 0.25)
    with pytest.raises(ValueError, match="pixel_pitch must be positive"):
        svc.validate_request(_req(1, pitch=(0.1, 0.0)), base, 0.25)
    with pytest.raises(ValueError, match="encoding must be raw8"):
        svc.validate_request(_req(1, enc=5), base, 0.25)
    plane, cfg = svc.validate_request(_req(1, (1, 2, 3, 1.0005, 0, 0, 0)), base, 0.25)
    assert cfg is base
    assert plane.pose.rotation.w == 1.0  # normalised (service.py:312)
    assert (plane.width, plane.height) == (24, 17)


def test_clamped_config_ranges():
    base = ResliceConfig(interp_radius=0.25)
    c = svc.clamped_config({"interp_radius": 100.0, "normal_threshold_deg": 95.0, "k_dist": -3.0}, base, 0.25)
    assert c.interp_radius == 8.0 * 0.25  # test_service.py:125 radius clamped to 8 voxels
    assert c.normal_threshold_deg == 89.9 and c.k_dist == 0.0
    assert c.inplane_threshold_deg == base.inplane_threshold_deg
    c = svc.clamped_config({"interp_radius": 1e-6, "inplane_threshold_deg": 0.0, "k_normal": 5e3}, base, 0.25)
    assert c.interp_radius == 0.05 * 0.25 and c.inplane_threshold_deg == 0.1 and c.k_normal == 1e3


def test_pack_coverage_and_payload():
    rng = np.random.default_rng(3)
    cov = rng.random((7, 13)) < 0.5
    assert svc.pack_coverage(cov) == np.packbits(cov, axis=None).tobytes()
    px = rng.integers(0, 256, (5, 6), dtype=np.uint8)
    assert svc.encode_image_payload(px, svc.ENCODING_RAW8) == px.tobytes()
    import zlib

    assert zlib.decompress(svc.encode_image_payload(px, svc.ENCODING_ZLIB)) == px.tobytes()


def test_flush_requests_newest_wins():
    class Fake:
        def process_request(self, msg):
            return svc.ResliceResponse(msg.request_id, svc.STATUS_OK, 1.0)

    out = svc.flush_requests([_req(4), _req(5), _req(9)], Fake())
    assert [r.status for r in out] == [svc.STATUS_SUPERSEDED, svc.STATUS_SUPERSEDED, svc.STATUS_OK]
    assert [r.superseded_by for r in out[:2]] == [9, 9] and out[2].request_id == 9
    assert svc.flush_requests([], Fake()) == []


# ---- GPU: packed coverage and batching --------------------------------------------------------

def _volume(rng, n=30000, extent=8.0, voxel=0.25):
    b = db.VolumeBuilder(db.BoundingBox((0, 0, 0), (extent,) * 3), voxel)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1.0
    b.insert_batch(rng.uniform(0, extent, (n, 3)), q, rng.integers(0, 256, n))
    return b.seal()


def _pose7(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    if q[0] < 0:
        q = -q
    t = rng.uniform(1.0, 7.0, 3)
    return (*t, *q)


@pytest.mark.gpu
def test_reslice_packed_equals_reslice_and_packbits(rng):
    vol = _volume(rng)
    cfg = ResliceConfig(interp_radius=0.5, normal_threshold_deg=80, inplane_threshold_deg=80)
    planes = [ReslicePlane(Pose(Quaternion(*_pose7(rng)[3:]), rng.uniform(1, 7, 3)), 23, 19, (0.2, 0.2))
              for _ in range(5)]  # 437 pixels: not a multiple of 8
    px, bits, _ = svc.reslice_packed(vol, planes, cfg)
    assert bits.shape == (5, (23 * 19 + 7) // 8)
    for k, p in enumerate(planes):
        one = db.reslice(vol, p, cfg)
        np.testing.assert_array_equal(px[k], one.pixels)
        assert bits[k].tobytes() == np.packbits(one.coverage, axis=None).tobytes()
        ref = oracle.reslice(vol, oracle.plane_params(p), oracle.cfg_array(cfg), p.width, p.height)
        np.testing.assert_array_equal(px[k], ref[0])


@pytest.mark.gpu
def test_batcher_concurrent_requests_match_library(rng):
    vol = _volume(rng)
    base = ResliceConfig(interp_radius=0.5, normal_threshold_deg=80, inplane_threshold_deg=80)
    reqs = []
    for i in range(48):
        cfgd = {"k_dist": 1.0} if i % 3 == 0 else None
        w, h = (24, 17) if i % 4 else (31, 9)
        reqs.append(_req(i, _pose7(rng), w, h, (0.2, 0.25), i % 2, cfgd))
    reqs.append(_req(99, (0, 0, 0, 3.0, 0, 0, 0)))  # invalid: answered with an error, others unaffected
    results = {}
    with svc.ResliceBatcher(vol, base, max_batch=8) as batcher:
        def worker(chunk):
            futs = [(r, batcher.submit(r)) for r in chunk]
            for r, f in futs:
                results[r.request_id] = f.result()

        threads = [threading.Thread(target=worker, args=(reqs[j::4],)) for j in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert batcher.requests == 48 and 1 <= batcher.launches <= 48
    bad = results.pop(99)
    assert bad.status == svc.STATUS_ERROR and "unit quaternion" in bad.message
    import zlib

    for r in reqs[:-1]:
        res = results[r.request_id]
        assert res.status == svc.STATUS_OK and (res.width, res.height) == (r.width, r.height)
        plane, cfg = svc.validate_request(r, base, vol.voxel_size)
        one = db.reslice(vol, plane, cfg)
        img = zlib.decompress(res.image) if r.encoding == 1 else res.image
        assert img == one.pixels.tobytes()
        assert res.coverage == np.packbits(one.coverage, axis=None).tobytes()


@pytest.mark.gpu
def test_batcher_serves_trilinear(rng):
    n, h, w = 12, 20, 22
    poses = [Pose(Quaternion.from_axis_angle((1, 0, 0), 0.01 * k), (0.0, 0.0, 0.1 * k)) for k in range(n)]
    ts = np.arange(n) / 30.0
    sweep = db.SweepRecording(rng.integers(0, 256, (n, h, w), dtype=np.uint8), ts, ts, poses, (0.1, 0.1))
    s = db.fill_holes(db.compound(sweep, voxel_size=0.125, margin=0.3), 3)
    reqs = [_req(i, (0.2, 0.3, 0.2 + 0.05 * i, 1.0, 0.0, 0.0, 0.0), 18, 15, (0.1, 0.1)) for i in range(10)]
    with svc.ResliceBatcher(s, max_batch=4) as batcher:
        futs = [batcher.submit(r) for r in reqs]
        out = [f.result() for f in futs]
        assert not batcher.directional
    for r, res in zip(reqs, out):
        plane, _ = svc.validate_request(r, ResliceConfig(), s.voxel_size)
        one = db.reslice_trilinear(s, plane)
        assert res.status == svc.STATUS_OK
        assert res.image == one.pixels.tobytes()
        assert res.coverage == np.packbits(one.coverage, axis=None).tobytes()


@pytest.mark.gpu
def test_reslice_packed_large_batch_unstaged(rng):
    """> 4 MB of output: the unstaged host-buffer path (direct copies) of dare_reslice_packed."""
    vol = _volume(rng, n=20000)
    cfg = ResliceConfig(interp_radius=0.5, normal_threshold_deg=80, inplane_threshold_deg=80)
    planes = [ReslicePlane(Pose(Quaternion(*_pose7(rng)[3:]), rng.uniform(1, 7, 3)), 256, 256, (0.03, 0.03))
              for _ in range(70)]
    px, bits, _ = svc.reslice_packed(vol, planes, cfg)
    ref_px, ref_cov, _ = db.reslice_batch(vol, planes, cfg)
    np.testing.assert_array_equal(px, ref_px)
    for k in range(len(planes)):
        assert bits[k].tobytes() == np.packbits(ref_cov[k], axis=None).tobytes()
