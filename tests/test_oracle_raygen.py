"""Pins for the oracle's ray generation (Eq. 19; spinning S:460-468; rosette R20).

Every expectation here comes from a closed form or an identity of rotations, not from the
oracle's own formula."""
import math

import numpy as np
import pytest

import synth


def _ident(t=(0.0, 0.0, 0.0)):
    return synth.pose(t)[None]


def test_forward_beam_identity(orc):
    # e = 0, a = 0, identity pose -> (1, 0, 0)   [S:466]
    o, d = orc.spinning_rays(np.array([0.0], np.float32), 1, 0.0, _ident((1.0, 2.0, 3.0)))
    assert np.allclose(d[0], [1, 0, 0], atol=1e-15)
    assert np.array_equal(o[0], [1.0, 2.0, 3.0])  # x_s := t_s


def test_zenith_beam(orc):
    # e = 90 deg -> (0, 0, 1)   [S:467]
    _, d = orc.spinning_rays(np.array([90.0], np.float32), 7, 0.0, _ident())
    assert np.allclose(d, [[0, 0, 1]] * 7, atol=1e-15)


def test_compass_quadrature(orc):
    # 1 channel, 4 columns, elevation 0 -> the four compass vectors, counter-clockwise from +x [S:458]
    _, d = orc.spinning_rays(np.array([0.0], np.float32), 4, 0.0, _ident())
    assert np.allclose(d, [[1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]], atol=1e-15)


def test_counts_and_layout(orc):
    # N_r = C x A and ray g = c*A + a (row-major)
    for name, cols, n in (("HDL64", 1800, 115200), ("OS128", 1024, 131072)):
        p = synth.spinning_preset(name, cols)
        o, d = orc.spinning_rays(p.elev_deg, p.columns, 0.0, _ident())
        assert d.shape == (n, 3)
    p = synth.spinning_preset("VLP16", 360)
    _, d = orc.spinning_rays(p.elev_deg, 360, 0.0, _ident())
    e = np.degrees(np.arcsin(d[:, 2])).reshape(16, 360)
    assert np.allclose(e, p.elev_deg.astype(np.float64)[:, None], atol=1e-9)
    az = np.degrees(np.arctan2(d[:, 1], d[:, 0])).reshape(16, 360) % 360.0
    assert np.allclose(az, np.arange(360)[None, :] * 1.0, atol=1e-9)


def test_yaw_equals_azimuth_offset(orc):
    # identity of rotations: Rz(psi) d(e, theta) = d(e, theta + psi)
    p = synth.spinning_preset("VLP16", 90)
    for psi in (0.3, -2.0, 3.0):
        _, d1 = orc.spinning_rays(p.elev_deg, 90, 0.0, synth.pose((0, 0, 0), yaw=psi)[None])
        _, d2 = orc.spinning_rays(p.elev_deg, 90, math.degrees(psi), _ident())
        assert np.max(np.abs(d1 - d2)) < 3e-7  # the pose matrix is float32-rounded


def test_pitch_shifts_elevation(orc):
    # Ry(p) (cos e, 0, sin e) = (cos(e - p), 0, sin(e - p))
    e = np.array([-20.0, -5.0, 0.0, 10.0], np.float32)
    pitch = math.radians(7.0)
    _, d = orc.spinning_rays(e, 1, 0.0, synth.pose((0, 0, 0), pitch=pitch)[None])
    exp = np.radians(e.astype(np.float64)) - pitch
    assert np.allclose(d, np.stack([np.cos(exp), 0 * exp, np.sin(exp)], 1), atol=3e-7)


def test_unit_norm_random_poses(orc):
    p = synth.spinning_preset("HDL64", 64)
    P = synth.random_poses(5, 1, (-50, -50, -5), (50, 50, 5))
    o, d = orc.spinning_rays(p.elev_deg, 64, 1.5, P)
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)
    assert np.array_equal(o.reshape(5, -1, 3)[:, 0], P[:, :, 3].astype(np.float64))


# ---- rosette -------------------------------------------------------------------------------
def test_rosette_sample_zero(orc):
    # n = 0, phase2_0 = 0: phi1 = phi2 = 0 -> delta = (Phi, 0) -> d = (cos Phi, sin Phi, 0)
    Phi = math.radians(35.2)
    _, d = orc.rosette_rays(4, 2611340, 1668595, 0, 35.2, _ident())
    assert np.allclose(d[0], [math.cos(Phi), math.sin(Phi), 0.0], atol=1e-15)


def test_rosette_opposed_phases_point_forward(orc):
    # inc1 = 2^31 (half a turn per sample), inc2 = 0: sample 1 has phi1 = 1/2, phi2 = 0 -> delta = 0
    _, d = orc.rosette_rays(2, 2 ** 31, 0, 0, 35.2, _ident())
    assert np.allclose(d[1], [1, 0, 0], atol=1e-15)
    # quarter turn: phi1 = 1/4 -> delta = Phi/2 (1, 1), |delta| = Phi / sqrt 2
    Phi = math.radians(35.2)
    _, d = orc.rosette_rays(2, 2 ** 30, 0, 0, 35.2, _ident())
    r = Phi / math.sqrt(2)
    s = math.sin(r) / r
    assert np.allclose(d[1], [math.cos(r), Phi / 2 * s, Phi / 2 * s], atol=1e-15)


def test_rosette_integer_phase_has_no_drift(orc):
    # period-4 phases repeat bit-for-bit at any sample index (exact 32-bit phase arithmetic)
    P = np.stack([synth.pose((0, 0, 0))] * 2)
    _, d = orc.rosette_rays(8, 2 ** 30, 3 * 2 ** 30, 12345, 35.2, P, first_frame=10 ** 9)
    d = d.reshape(2, 8, 3)
    assert np.array_equal(d[0, :4], d[0, 4:])
    assert np.array_equal(d[0], d[1])
    _, d0 = orc.rosette_rays(8, 2 ** 30, 3 * 2 ** 30, 12345, 35.2, synth.pose((0, 0, 0))[None], first_frame=0)
    assert np.array_equal(d0, d[0])


def test_rosette_cone_and_nonrepetition(orc):
    ros = synth.rosette_default()
    P = np.stack([synth.pose((0, 0, 0))] * 3)
    _, d = orc.rosette_rays(ros.points_per_frame, ros.inc1, ros.inc2, ros.phase2_0, ros.half_fov_deg, P)
    ang = np.degrees(np.arccos(np.clip(d[:, 0], -1, 1)))
    assert ang.max() <= 35.2 + 1e-9
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)
    f = d.reshape(3, -1, 3)
    assert np.mean(np.all(np.isclose(f[0], f[1]), axis=1)) < 0.01  # frames do not repeat


def test_pattern_dispatch(orc):
    cfg = synth.config("C1")
    o, d = orc.pattern_rays(cfg["pattern"], cfg["poses"])
    assert d.shape == (16 * 360, 3)
