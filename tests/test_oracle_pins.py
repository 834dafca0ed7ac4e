"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Every check compares the oracle with something other than itself: closed forms,
independent libraries (scipy Rotation/Slerp, scipy real SH, numpy cumsum, Monte Carlo),
brute force on tiny inputs, hand-worked golden fixtures (tests/golden/) and invariants.
Citations: P:n = PAPER.md line n; S:n = SPEC.md line n (test ideas only).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation, Slerp

from paper_2510_12901_b200 import synth as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def qmul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def ident_pose(t=(0.0, 0.0, 0.0)):
    return np.array([1.0, 0, 0, 0, *t])


# ---------------------------------------------------------------- O1 covariance
def test_covariance_closed_forms(oracle_mod):
    O = oracle_mod
    assert np.allclose(O.covariance([1, 0, 0, 0], [1, 1, 1]), np.eye(3), atol=1e-15)
    assert np.allclose(O.covariance([1, 0, 0, 0], [2, 1, 1]), np.diag([4, 1, 1]), atol=1e-15)
    q90 = [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)]
    assert np.allclose(O.covariance(q90, [2, 1, 1]), np.diag([1, 4, 1]), atol=1e-12)


def test_rotation_matches_scipy_and_equivariance(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(0)
    for _ in range(50):
        q = rng.normal(size=4)
        R = O.quat_to_rot(q)
        Rs = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy: scalar-last
        assert np.allclose(R, Rs, atol=1e-12)
        q1 = rng.normal(size=4)
        q1 /= np.linalg.norm(q1)
        s = rng.uniform(0.1, 2, 3)
        lhs = O.covariance(qmul(q1, q / np.linalg.norm(q)), s)
        R1 = O.quat_to_rot(q1)
        assert np.allclose(lhs, R1 @ O.covariance(q, s) @ R1.T, atol=1e-10)
        assert np.allclose(np.sort(np.linalg.eigvalsh(O.covariance(q, s))), np.sort(s ** 2), atol=1e-10)


# ---------------------------------------------------------------- O2 sigma points / UT
@pytest.mark.parametrize("ut", [(1.0, 2.0, 0.0), (0.5, 2.0, 1.0), (1.0, 0.0, 2.0)])
def test_sigma_points_reproduce_moments(oracle_mod, ut):
    O = oracle_mod
    rng = np.random.default_rng(1)
    for _ in range(20):
        mu, q, s = rng.normal(size=3) * 5, rng.normal(size=4), rng.uniform(0.01, 1.0, 3)
        pts, wm, wc = O.sigma_points(mu, q, s, ut)
        assert pts.shape == (7, 3)
        assert abs(wm.sum() - 1.0) < 1e-12
        mean = (wm[:, None] * pts).sum(0)
        cov = sum(wc[i] * np.outer(pts[i] - mu, pts[i] - mu) for i in range(7))
        assert np.allclose(mean, mu, atol=1e-12)
        assert np.allclose(cov, O.covariance(q, s), atol=1e-12)


@pytest.mark.parametrize("ut", [(1.0, 2.0, 0.0), (0.7, 2.0, 0.5)])
def test_ut_exact_for_affine_sensor(oracle_mod, ut):
    """north star: the UT of a linear projection equals the exact projected covariance."""
    O = oracle_mod
    rng = np.random.default_rng(2)
    for _ in range(50):
        mu, q, s = rng.normal(size=3) * 3, rng.normal(size=4), rng.uniform(0.01, 2.0, 3)
        A, b = rng.normal(size=(2, 3)), rng.normal(size=2)
        mean, cov = O.ut_affine(mu, q, s, A, b, ut)
        Sig = O.covariance(q, s)
        assert np.allclose(mean, A @ mu + b, atol=1e-12)
        assert np.allclose(cov, A @ Sig @ A.T, atol=1e-12)


def test_ut_lidar_monte_carlo(oracle_mod):
    """UT conic of Eq. 3 vs 1e5 samples through atan2/asin: within 2% Frobenius."""
    O = oracle_mod
    cfg = S.lidar_config("A")
    rng = np.random.default_rng(3)
    cases = [((10.0, 0, 0), (0.3, 0.3, 0.3)), ((0, 10.0, 1.0), (0.5, 0.2, 0.1)), ((-5.0, 3.0, -1.0), (0.4, 0.1, 0.6))]
    for mu, s in cases:
        q = rng.normal(size=4)
        scene = {"means": np.array([mu], np.float32), "quats": np.array([q], np.float32),
                 "scales": np.array([s], np.float32), "opacity": np.array([0.9], np.float32),
                 "sh": np.zeros((1, 16, 3), np.float32)}
        p0 = S.pose([1, 0, 0, 0], [0, 0, 0])
        proj = O.project_lidar(scene, cfg, p0, p0, K=0)
        Sig = O.covariance(q, np.asarray(s, np.float32).astype(np.float64))
        x = rng.multivariate_normal(np.asarray(mu, np.float32).astype(np.float64), Sig, 100000)
        r = np.linalg.norm(x, axis=1)
        ang = np.stack([np.arctan2(x[:, 1], x[:, 0]), np.arcsin(x[:, 2] / r)], 1)
        C = np.cov(ang.T)
        ut = proj["cov2d"][0]
        Cu = np.array([[ut[0], ut[1]], [ut[1], ut[2]]])
        assert np.linalg.norm(Cu - C) / np.linalg.norm(C) < 0.02
        assert np.allclose(proj["mean2d"][0], ang.mean(0), atol=3 * np.sqrt(np.diag(C)).max() / 100)


# ---------------------------------------------------------------- O3 poses (A4)
def test_pose_interpolation(oracle_mod):
    O = oracle_mod
    p = np.array([0.9, 0.1, -0.2, 0.3, 1.0, 2.0, 3.0])
    for s in (0.0, 0.3, 1.0):
        R, t = O.pose_at(p, p, s)
        assert np.array_equal(R, O.quat_to_rot(p[:4])) and np.array_equal(t, p[4:])
    a, b = ident_pose((0, 0, 0)), ident_pose((1.0, 0, 0))  # 10 m/s over 0.1 s
    assert np.allclose(O.pose_at(a, b, 1.0)[1], [1.0, 0, 0]) and np.allclose(O.pose_at(a, b, 0.5)[1], [0.5, 0, 0])
    yaw90 = np.array([math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4), 0, 0, 0])
    R, _ = O.pose_at(ident_pose(), yaw90, 0.5)
    assert np.allclose(R, Rotation.from_euler("z", 45, degrees=True).as_matrix(), atol=1e-12)
    rng = np.random.default_rng(4)
    for _ in range(20):
        q0, q1 = rng.normal(size=4), rng.normal(size=4)
        q0 /= np.linalg.norm(q0)
        q1 /= np.linalg.norm(q1)
        sl = Slerp([0, 1], Rotation.from_quat([[*q0[1:], q0[0]], [*q1[1:], q1[0]]]))
        for s in (0.25, 0.5, 0.9):
            R, _ = O.pose_at(np.r_[q0, 0, 0, 0], np.r_[q1, 0, 0, 0], s)
            assert np.allclose(R, sl([s]).as_matrix()[0], atol=1e-10)


# ---------------------------------------------------------------- O4 Eq. 3 + rolling shutter
def test_eq3_axis_points(oracle_mod):
    O = oracle_mod
    cfg = S.lidar_config("A")
    p = ident_pose()
    assert np.allclose(O.lidar_point([1, 0, 0], cfg, p, p, 0)[:3], [0, 0, 1], atol=1e-15)
    assert np.allclose(O.lidar_point([0, 1, 0], cfg, p, p, 0)[:3], [math.pi / 2, 0, 1], atol=1e-15)
    assert np.allclose(O.lidar_point([0, 0, 1], cfg, p, p, 0)[:3], [0, math.pi / 2, 1], atol=1e-15)


def test_rolling_shutter_static_bitwise_and_fixed_point(oracle_mod):
    from scipy.optimize import brentq
    O = oracle_mod
    cfg = S.lidar_config("A")
    p = np.array([0.98, 0.0, 0.05, 0.2, 0.3, -0.1, 1.8])
    x = np.array([7.0, -3.0, 0.5])
    a = O.lidar_point(x, cfg, p, p, 0)
    for K in (1, 2, 5):
        b = O.lidar_point(x, cfg, p, p, K)
        assert np.array_equal(a[:3], b[:3])
    # linear motion along +y at 5 m per revolution; point at (10, 0, 0): phi(s) = atan2(-5 s, 10)
    p0, p1 = ident_pose((0, 0, 0)), ident_pose((0, 5.0, 0))
    a0 = float(np.float32(cfg.azimuth_start))  # the ABI's float32 phi_start
    f = lambda s: (math.atan2(-5.0 * s, 10.0) - a0) / (2 * math.pi) - s  # noqa: E731
    s_star = brentq(f, 0.0, 1.0, xtol=1e-15)
    errs = [abs(O.lidar_point([10, 0, 0], cfg, p0, p1, K)[3] - s_star) for K in range(1, 14)]
    assert errs[-1] < 1e-9
    assert all(e2 <= e1 * 0.2 + 1e-15 for e1, e2 in zip(errs, errs[1:]))  # geometric contraction


def test_seam_continuity(oracle_mod):
    """A Gaussian swept across phi = pi (co-rotating with its azimuth, so by symmetry about
    z its conic must stay the same) keeps a continuous conic and box."""
    O = oracle_mod
    cfg = S.lidar_config("A")
    p = S.pose([1, 0, 0, 0], [0, 0, 0])
    angs = np.linspace(math.pi - 0.02, math.pi + 0.02, 81)
    means = np.stack([10 * np.cos(angs), 10 * np.sin(angs), np.full_like(angs, 1.0)], 1)
    base = np.array([0.9, 0.1, 0.2, 0.3])
    quats = np.array([qmul([math.cos(a / 2), 0, 0, math.sin(a / 2)], base) for a in angs])
    n = len(angs)
    scene = {"means": means.astype(np.float32), "quats": quats.astype(np.float32),
             "scales": np.tile(np.array([[0.3, 0.1, 0.2]], np.float32), (n, 1)),
             "opacity": np.full(n, 0.5, np.float32), "sh": np.zeros((n, 16, 3), np.float32)}
    proj = O.project_lidar(scene, cfg, p, p, K=0)
    cov = proj["cov2d"]
    assert np.abs(cov - cov[0]).max() < 1e-5 * np.abs(cov).max()  # float32 inputs -> ~1e-7 rel.
    width = proj["box"][:, 1].astype(np.float64) - proj["box"][:, 0]
    assert np.abs(width - width[0]).max() < 1e-6
    assert ((proj["mean2d"][:, 0] >= -math.pi) & (proj["mean2d"][:, 0] < math.pi)).all()
    mean_unwrapped = np.unwrap(proj["mean2d"][:, 0])
    off = mean_unwrapped - angs  # constant UT bias (w_m0 = 0), no jump at the seam
    assert np.abs(off - off[0]).max() < 1e-6 and abs(off[0]) < 1e-3


# ---------------------------------------------------------------- O9 SH
def _real_sh_scipy(l, m, theta, phi):
    from scipy.special import sph_harm_y
    if m == 0:
        return sph_harm_y(l, 0, theta, phi).real
    y = sph_harm_y(l, abs(m), theta, phi)
    return math.sqrt(2) * (-1) ** m * (y.imag if m < 0 else y.real)


def test_sh_basis_orthonormal_and_scipy(oracle_mod):
    O = oracle_mod
    # quadrature over the sphere: Gauss-Legendre in cos(theta) x uniform phi
    xg, wg = np.polynomial.legendre.leggauss(24)
    phis = np.linspace(0, 2 * np.pi, 48, endpoint=False)
    B, W = [], []
    for ct, w in zip(xg, wg):
        st = math.sqrt(1 - ct * ct)
        for ph in phis:
            d = np.array([st * math.cos(ph), st * math.sin(ph), ct])
            row = []
            for k in range(16):
                sh = np.zeros((16, 3))
                sh[k, 0] = 1.0
                row.append(O.sh_eval(sh, d)[0])
            B.append(row)
            W.append(w * 2 * np.pi / len(phis))
    B, W = np.array(B), np.array(W)
    G = (B * W[:, None]).T @ B
    assert np.allclose(G, np.eye(16), atol=1e-10)
    # each basis function equals +-(scipy real SH) of its degree (3DGS sign convention)
    rng = np.random.default_rng(5)
    lm = [(0, 0)] + [(1, m) for m in (-1, 0, 1)] + [(2, m) for m in range(-2, 3)] + [(3, m) for m in range(-3, 4)]
    dirs = rng.normal(size=(20, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    for k, (l, m) in enumerate(lm):
        ours, ref = [], []
        for d in dirs:
            sh = np.zeros((16, 3))
            sh[k, 0] = 1.0
            ours.append(O.sh_eval(sh, d)[0])
            ref.append(_real_sh_scipy(l, m, math.acos(d[2]), math.atan2(d[1], d[0])))
        ours, ref = np.array(ours), np.array(ref)
        sgn = np.sign(np.dot(ours, ref))
        assert np.allclose(ours, sgn * ref, atol=1e-12), (l, m)


def test_sh_dc_parity_linearity(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(6)
    sh = np.zeros((16, 3))
    sh[0] = [1.0, 2.0, -3.0]
    for _ in range(5):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        assert np.allclose(O.sh_eval(sh, d), np.array([1, 2, -3]) * 0.2820947918, atol=1e-10)
    z = np.zeros((16, 3))
    z[2, 0] = 1.0  # degree-1 z coefficient
    assert np.isclose(O.sh_eval(z, [0, 0, 1])[0], -O.sh_eval(z, [0, 0, -1])[0])
    a, b = rng.normal(size=(16, 3)), rng.normal(size=(16, 3))
    d = np.array([0.3, -0.5, 0.81])
    d /= np.linalg.norm(d)
    assert np.allclose(O.sh_eval(2 * a - 3 * b, d), 2 * O.sh_eval(a, d) - 3 * O.sh_eval(b, d), atol=1e-12)


# ---------------------------------------------------------------- O12 response
def _mrows(q, s):
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    return (R.T / np.asarray(s)[:, None]).reshape(-1)


def test_response_closed_forms(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(7)
    for _ in range(200):
        mu = rng.normal(size=3) * 10
        q, s = rng.normal(size=4), rng.uniform(0.05, 2.0, 3)
        o = rng.normal(size=3)
        d = mu - o
        d /= np.linalg.norm(d)
        tau, d2 = O.response(mu, _mrows(q, s), o, d)  # ray through the mean
        assert abs(tau - np.linalg.norm(mu - o)) < 1e-9 and abs(d2) < 1e-12
        # analytic tau_max = d^T Sigma^-1 (mu - o) / d^T Sigma^-1 d ; delta^2 = min Mahalanobis
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        Sinv = np.linalg.inv(O.covariance(q, s))
        tau_a = d @ Sinv @ (mu - o) / (d @ Sinv @ d)
        x = o + tau_a * d - mu
        tau, d2 = O.response(mu, _mrows(q, s), o, d)
        assert abs(tau - tau_a) < 1e-8 * (1 + abs(tau_a))
        assert abs(d2 - x @ Sinv @ x) < 1e-8 * (1 + d2)
    # isotropic: tau = (mu - o).d ; unit Mahalanobis -> exp(-1/2)
    mu, o, d = np.array([5.0, 1.0, 0.0]), np.zeros(3), np.array([1.0, 0, 0])
    tau, d2 = O.response(mu, _mrows([1, 0, 0, 0], [1, 1, 1]), o, d)
    assert tau == pytest.approx(5.0) and d2 == pytest.approx(1.0) and math.exp(-d2 / 2) == pytest.approx(0.60653066)


def test_response_dense_scan(oracle_mod):
    """argmax of rho along the ray from a 1e4-step scan agrees within one step."""
    O = oracle_mod
    rng = np.random.default_rng(8)
    for _ in range(50):
        mu = rng.normal(size=3) * 3 + np.array([6.0, 0, 0])
        q, s = rng.normal(size=4), rng.uniform(0.1, 1.0, 3)
        o, d = np.zeros(3), rng.normal(size=3) * 0.2 + np.array([1.0, 0, 0])
        d /= np.linalg.norm(d)
        Sinv = np.linalg.inv(O.covariance(q, s))
        taus = np.linspace(0, 15, 10001)
        X = o[None] + taus[:, None] * d[None] - mu[None]
        m = np.einsum("ni,ij,nj->n", X, Sinv, X)
        tau, d2 = O.response(mu, _mrows(q, s), o, d)
        assert abs(taus[np.argmin(m)] - tau) <= (taus[1] - taus[0]) * 1.01 or tau < 0 or tau > 15
        assert d2 <= m.min() + 1e-9


# ---------------------------------------------------------------- O12 compositing
def _one_ray(O, mus, sigmas, feats, s=0.05, near=0.1, alpha_max=0.99, T_min=1e-4, alpha_min=1 / 255):
    n = len(mus)
    rec = {"mu": np.array(mus, float), "Mrows": np.tile(_mrows([1, 0, 0, 0], [s, s, s]), (n, 1)),
           "sigma": np.array(sigmas, float), "feat": np.array(feats, float),
           "box": np.tile(np.array([[-1, 1, -1, 1]], np.float32), (n, 1))}
    keys = np.array([np.linalg.norm(m) for m in mus], np.float32)
    ids, ranges = O.sort_all(np.ones(n, np.int32), keys)
    od = np.array([[0, 0, 0, 1.0, 0, 0]])
    return O.composite(rec, ids, ranges, np.zeros(1, np.int32), np.zeros(1, np.float32), np.zeros(1, np.float32),
                       od, wrap=1, near=near, alpha_max=alpha_max, T_min=T_min, alpha_min=alpha_min)


def test_composite_worked_examples(oracle_mod):
    O = oracle_mod
    out = _one_ray(O, [[4.0, 0, 0]], [0.8], [[1, 1, 1]])
    assert out["opacity"][0] == pytest.approx(0.8) and out["depth"][0] == pytest.approx(4.0)
    out = _one_ray(O, [[5.0, 0, 0], [2.0, 0, 0]], [0.5, 0.5], [[1, 0, 0], [1, 0, 0]])
    assert out["opacity"][0] == pytest.approx(0.75) and out["depth"][0] == pytest.approx(3.0)
    empty = _one_ray(O, [[5.0, 0, 0]], [0.5], [[0, 0, 0]], near=100.0)  # nothing in front -> no return
    g, bd = O.decode_lidar(empty["feat"])
    assert empty["opacity"][0] == 0 and bd[0] == pytest.approx(0.5)


def test_composite_conservation_and_termination(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(9)
    for trial in range(20):
        n = 60
        mus = np.stack([rng.uniform(1, 30, n), rng.normal(0, 0.03, n), rng.normal(0, 0.03, n)], 1)
        sig = rng.uniform(0.05, 0.99, n)
        out = _one_ray(O, mus, sig, np.ones((n, 3)))
        assert out["opacity"][0] + out["T_final"][0] == pytest.approx(1.0, abs=1e-12)
        assert out["opacity"][0] <= 1.0
        out0 = _one_ray(O, mus, sig, np.ones((n, 3)), T_min=0.0)
        assert abs(out0["opacity"][0] - out["opacity"][0]) < 1e-3
        # T monotone: removing the tail can only raise T
        outh = _one_ray(O, mus[np.argsort(np.linalg.norm(mus, axis=1))][: n // 2],
                        sig[np.argsort(np.linalg.norm(mus, axis=1))][: n // 2], np.ones((n // 2, 3)), T_min=0.0)
        assert outh["T_final"][0] >= out0["T_final"][0] - 1e-15


def test_decode_closed_forms(oracle_mod):
    O = oracle_mod
    g, bd = O.decode_lidar(np.array([[0.3, math.log(3.0), 0.0], [0.5, 1.7, 1.7], [0, 50.0, -50.0], [0, -50.0, 50.0]]))
    assert g[0] == 0.3 and bd[0] == pytest.approx(0.25) and bd[1] == pytest.approx(0.5)
    assert np.isfinite(bd).all() and bd[2] < 1e-40 and bd[3] == pytest.approx(1.0)


def test_opaque_wall_depth(oracle_mod):
    """Opaque wall of particles at 10 m -> hit rays return 10 m within 0.05 m."""
    O = oracle_mod
    cfg = S.lidar_config("A")
    ys, zs = np.meshgrid(np.arange(-8, 8, 0.1), np.arange(-3.0, 4.0, 0.1))
    n = ys.size
    scene = {"means": np.stack([np.full(n, 10.0), ys.ravel(), zs.ravel()], 1).astype(np.float32),
             "quats": np.tile(np.array([[1, 0, 0, 0]], np.float32), (n, 1)),
             "scales": np.tile(np.array([[0.01, 0.08, 0.08]], np.float32), (n, 1)),
             "opacity": np.full(n, 0.99, np.float32), "sh": np.zeros((n, 16, 3), np.float32)}
    p = S.pose([1, 0, 0, 0], [0, 0, 0])
    out = O.render_lidar(scene, cfg, pose0=p, pose1=p)
    od = out["ray_od"]
    hit = out["opacity"] > 0.99
    assert hit.sum() > 50
    expect = 10.0 / od[hit, 3]  # plane x = 10 along each ray
    assert np.abs(out["depth"][hit] - expect).max() < 0.05


def _scaled_scene(scene, f):
    out = dict(scene)
    out["means"] = scene["means"] * np.float32(f)
    out["scales"] = scene["scales"] * np.float32(f)
    return out


@pytest.mark.parametrize("divergence", [0.0, 1.5e-3])
def test_whole_scan_scale_covariance(oracle_mod, divergence):
    """Whole LiDAR scan on a realistic scene (config-B sensor, rolling shutter, a 20k
    corridor subset): a scan is a function of lengths only through dimensionless ratios
    -- the sensor model (Eq. 3) sees directions, the canonical response and the
    beam-divergence covariance (App. C, theta^2 r^2) are homogeneous, the depth key (A19)
    orders by distance -- so scaling every length by 2 (means, scales, sensor track,
    minimum range; exact in binary floating point) must return depth x 2 and every other
    output bit for bit.  A term of the wrong dimension anywhere in O1-O13 (a dropped
    square, Sigma for Sigma^-1, an absolute epsilon) breaks it."""
    import copy
    O = oracle_mod
    cfg = S.lidar_config("B")
    cfg.beam_divergence = divergence
    scene = S.corridor_scene(7, 20000, x_range=(-30.0, 30.0))
    scene["means"] = (scene["means"] - np.float32([0.0, 0.0, 1.8])).astype(np.float32)  # sensor at the origin
    p0 = S.pose([1, 0, 0, 0], [0, 0, 0])
    ref = O.render_lidar(scene, cfg, pose0=p0, pose1=S.pose(S.yaw_quat(0.03), [1.0, 0.0, 0.0]))
    cfg2 = copy.deepcopy(cfg)
    cfg2.min_range = cfg.min_range * 2
    got = O.render_lidar(_scaled_scene(scene, 2), cfg2, pose0=p0, pose1=S.pose(S.yaw_quat(0.03), [2.0, 0.0, 0.0]))
    assert (ref["opacity"] > 0.5).mean() > 0.2 and (ref["n_contrib"] > 0).mean() > 0.3
    for k in ("depth", "depth_accum"):
        assert np.array_equal(got[k], 2 * ref[k]), k
    for k in ("feat", "opacity", "T_final", "n_contrib", "scanned", "inbox", "intensity", "raydrop"):
        assert np.array_equal(got[k], ref[k]), k
    assert np.array_equal(got["ray_od"][:, :3], 2 * ref["ray_od"][:, :3])
    assert np.array_equal(got["ray_od"][:, 3:], ref["ray_od"][:, 3:])


def test_whole_frame_scale_covariance(oracle_mod):
    """The same for a rolling-shutter KB-fisheye frame (D-small, a 20k camera corridor
    subset): projection is scale free (x/z, atan2(rho, z)), the near plane scales."""
    import copy
    O = oracle_mod
    cam = S.camera_config("D-small")
    scene = S.corridor_scene(8, 20000, x_range=(-5.0, 40.0), kind="camera", ego=(1.5, 0.0, 1.6))
    scene["means"] = (scene["means"] - np.float32([1.5, 0.0, 1.6])).astype(np.float32)
    c0 = S.pose(S.CAM_FORWARD_Q, [0, 0, 0])
    ref = O.render_camera(scene, cam, pose0=c0, pose1=S.pose(S.yaw_quat(0.009, S.CAM_FORWARD_Q), [0.3, 0, 0]))
    cam2 = copy.deepcopy(cam)
    cam2.near = cam.near * 2
    got = O.render_camera(_scaled_scene(scene, 2), cam2, pose0=c0,
                          pose1=S.pose(S.yaw_quat(0.009, S.CAM_FORWARD_Q), [0.6, 0, 0]))
    assert (ref["opacity"] > 0.2).mean() > 0.1
    for k in ("depth", "depth_accum"):
        assert np.array_equal(got[k], 2 * ref[k]), k
    for k in ("feat", "opacity", "T_final", "n_contrib", "scanned", "inbox"):
        assert np.array_equal(got[k], ref[k]), k


# ---------------------------------------------------------------- O7 tiling
def _tiling_for(beams_rad, A, n_phi, M, cull_az=1600):
    cfg = S.LidarConfig("t", np.asarray(beams_rad, np.float32), A, n_phi=n_phi, max_rays_per_tile=M,
                        cull_az_cells=cull_az)
    from oracle import oracle as O
    return O.Tiling(cfg)


def test_proc1_handworked_golden(oracle_mod):
    g = json.load(open(os.path.join(GOLDEN, "proc1_handworked.json")))
    t = _tiling_for(np.radians(np.array(g["elevations_deg"], np.float64)).astype(np.float32), g["n_azimuth"],
                    g["n_phi"], g["M"])
    assert t.n_phi == g["expect_n_phi"] and t.n_theta == g["expect_n_theta"]
    exp = np.radians(np.array(g["expect_bounds_deg"]))
    assert np.allclose(t.bounds, exp, atol=1e-7)
    assert (np.diff(t.tile_ray_offsets) == g["expect_rays_per_tile"]).all()
    assert list(t.ray_tile[: g["n_azimuth"]] % t.n_theta) == g["expect_ray_cols"]


def test_proc1_uniform_quartiles(oracle_mod):
    """64 uniform beams in [-25, 15] deg, N_phi=4 -> 16/16/16/16, boundaries in the
    gap between beams 15|16, 31|32, 47|48 (A8 reading of 'cross integer boundaries')."""
    beams = np.radians(np.linspace(-25.0, 15.0, 64)).astype(np.float32)
    t = _tiling_for(beams, 1800, 4, 32)
    assert t.n_phi == 4
    counts = np.bincount([t.elev_tile(float(b)) for b in beams], minlength=4)
    assert list(counts) == [16, 16, 16, 16]
    for k, (lo, hi) in enumerate([(15, 16), (31, 32), (47, 48)]):
        assert beams[lo] < t.bounds[k + 1] <= beams[hi]
        assert abs(float(t.bounds[k + 1]) - 0.5 * (float(beams[lo]) + float(beams[hi]))) < 1e-7
    assert t.n_theta == math.ceil(16 * 1800 / 32)


def test_proc1_skewed_and_invariants(oracle_mod):
    beams = np.radians(np.r_[np.linspace(-1.0, 3.0, 60, endpoint=False), np.linspace(3.0, 19.0, 4)]).astype(np.float32)
    t = _tiling_for(beams, 1800, 4, 32)
    inside = sum(1 for k in range(t.n_phi) if t.bounds[k] >= np.radians(-1.0) - 1e-7
                 and t.bounds[k + 1] <= np.radians(3.0) + 1e-7)
    assert inside >= 3
    rng = np.random.default_rng(10)
    for trial in range(40):
        B = int(rng.integers(1, 80))
        beams = np.sort(rng.uniform(-0.5, 0.3, B)).astype(np.float32)
        if trial % 5 == 0:
            beams = np.round(beams, 2).astype(np.float32)  # duplicates / shared bins
        A = int(rng.integers(16, 400))
        n_phi = int(rng.integers(1, 40))
        prev = None
        for M in (8, 16, 32, 64, 128, 256):
            t = _tiling_for(beams, A, n_phi, M)
            assert 1 <= t.n_phi <= n_phi and t.bounds.shape[0] <= n_phi + 1
            assert np.all(np.diff(t.bounds) > 0) or t.n_phi == 1
            assert t.tile_ray_offsets[-1] == B * A  # total occupancy = ray count
            beams_per = np.bincount([t.elev_tile(float(b)) for b in beams], minlength=t.n_phi)
            assert (beams_per > 0).all()  # no empty elevation tile
            assert t.n_theta == min(A, max(1, math.ceil(beams_per.max() * A / M)))
            if prev is not None:
                assert t.n_theta <= prev  # non-increasing in M
            prev = t.n_theta
            if beams_per.max() <= M and M % beams_per.max() == 0 and A % t.n_theta == 0:
                assert t.max_rays_in_tile <= M  # "count per tile under M"
        t2 = _tiling_for(beams, A, n_phi, 32)
        t3 = _tiling_for(beams, A, n_phi, 32)
        assert np.array_equal(t2.bounds, t3.bounds) and np.array_equal(t2.sat, t3.sat)  # bit-identical reruns


def test_tiling_paper_configs(oracle_mod):
    for name, exp in (("A", (8, 64, 32)), ("B", (16, 225, 32)), ("C", (16, 332, 32))):
        t = oracle_mod.Tiling(S.lidar_config(name))
        assert (t.n_phi, t.n_theta, t.max_rays_in_tile) == exp
        assert t.tile_ray_offsets[-1] == t.n_rays


# ---------------------------------------------------------------- SAT + culling
def test_sat_bruteforce(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(11)
    for _ in range(20):
        h, w = rng.integers(1, 64, 2)
        mask = (rng.uniform(size=(h, w)) < rng.uniform(0, 0.5)).astype(np.int32)
        sat = np.zeros((h + 1, w + 1), np.int32)
        sat[1:, 1:] = mask.cumsum(0).cumsum(1)
        for _ in range(50):
            r0, r1 = np.sort(rng.integers(0, h, 2))
            c0, c1 = np.sort(rng.integers(0, w, 2))
            assert O.sat_query(sat, r0, r1, c0, c1) == mask[r0:r1 + 1, c0:c1 + 1].sum()
    z = np.zeros((4, 4), np.int32)
    assert O.sat_query(z, 0, 2, 0, 2) == 0
    f = np.zeros((4, 4), np.int32)
    f[1:, 1:] = np.ones((3, 3)).cumsum(0).cumsum(1)
    assert O.sat_query(f, 0, 2, 0, 2) == 9


def test_oracle_sat_matches_mask(oracle_mod):
    t = oracle_mod.Tiling(S.lidar_config("B"))
    rows, cols = t.sat_rows - 1, t.sat_cols - 1
    mask = np.zeros((rows, cols), np.int32)
    mask[t.ray_cell_row, t.ray_cell_col] = 1
    ref = np.zeros_like(t.sat)
    ref[1:, 1:] = mask.cumsum(0).cumsum(1)
    assert np.array_equal(ref, t.sat)


def _membership(box, a, b, pi_f, two_pi_f):
    """Per-ray box membership (numpy float32 restatement of the O12 rule, for invariants);
    a, b are float32 arrays of ray azimuth / elevation."""
    lo, hi, lb, hb = [np.float32(x) for x in box]
    inb = (lb <= b) & (b <= hb)
    if np.float32(hi - lo) >= two_pi_f:
        return inb
    m = (lo <= a) & (a <= hi)
    if lo < -pi_f:
        m |= np.float32(lo + two_pi_f) <= a
    if hi > pi_f:
        m |= a <= np.float32(hi - two_pi_f)
    return inb & m


@pytest.mark.parametrize("config", ["A", "tiny"])
def test_culling_exact_and_rect_contains_members(oracle_mod, config):
    """Culled => no ray inside the box; every member ray's tile lies in the rect."""
    O = oracle_mod
    cfg = S.lidar_config(config)
    t = O.Tiling(cfg)
    scene = S.scene_for(config, seed=3)
    proj = O.project_lidar(scene, cfg)
    count, rect = O.cull_lidar(proj["valid"], proj["box"], t, True)
    count0, _ = O.cull_lidar(proj["valid"], proj["box"], t, False)
    assert (count <= count0).all()
    tiles_of = lambda g: {r * t.n_theta + (rect[g, 2] + c) % t.n_theta  # noqa: E731
                          for r in range(rect[g, 0], rect[g, 1] + 1) for c in range(rect[g, 3])}
    for g in np.nonzero(proj["valid"])[0][:300]:
        members = np.nonzero(_membership(proj["box"][g], t.ray_az, t.ray_el, t.pi_f, t.two_pi_f))[0]
        if count[g] == 0:
            assert len(members) == 0
        else:
            assert {int(t.ray_tile[r]) for r in members} <= tiles_of(g)


@pytest.mark.parametrize("config", ["A", "tiny", "B-small"])
def test_exact_culling_is_the_brute_force_tile_set(oracle_mod, config):
    """Exact ray-containment culling (A32): the tile set of every particle equals, by brute
    force over every ray, the set of render tiles holding a ray inside its box under the
    compositing membership rule (A12); it refines the paper's SAT culling (subset)."""
    O = oracle_mod
    if config == "B-small":  # Pandar64 beams, rolling shutter, a random subset of the corridor
        cfg = S.lidar_config("B")
        cfg.n_azimuth = 600
        scene = S.scene_for("B", n=3000)
    else:
        cfg = S.lidar_config(config)
        scene = S.scene_for(config, seed=5)
    t = O.Tiling(cfg)
    proj = O.project_lidar(scene, cfg)
    count2, rect2 = O.cull_lidar(proj["valid"], proj["box"], t, 2)
    count1, rect1 = O.cull_lidar(proj["valid"], proj["box"], t, 1)
    tiles = lambda rect, g: {r * t.n_theta + (rect[g, 2] + c) % t.n_theta  # noqa: E731
                             for r in range(rect[g, 0], rect[g, 1] + 1) for c in range(rect[g, 3])}
    n_checked = n_refined = 0
    for g in np.nonzero(proj["valid"])[0][:400]:
        members = np.nonzero(_membership(proj["box"][g], t.ray_az, t.ray_el, t.pi_f, t.two_pi_f))[0]
        brute = {int(t.ray_tile[r]) for r in members}
        got = tiles(rect2, g) if count2[g] else set()
        assert got == brute, g
        assert count2[g] == len(brute)
        assert count2[g] == 0 or brute <= tiles(rect1, g)
        n_checked += 1
        n_refined += count2[g] < count1[g]
    assert n_checked > 50 and n_refined > 0


def test_exact_culling_render_unchanged(oracle_mod):
    """Outputs do not depend on the culling mode (A12): off, SAT and exact (A32)."""
    O = oracle_mod
    cfg = S.lidar_config("A")
    scene = S.scene_for("A")
    outs = [O.render_lidar(scene, cfg, mode="tiled", enable_cull=m) for m in (0, 1, 2)]
    for o in outs[1:]:
        for k in ("feat", "opacity", "depth_accum", "T_final", "n_contrib"):
            assert np.array_equal(outs[0][k], o[k]), k


# ---------------------------------------------------------------- O13 tiled == brute force
def test_tiled_equals_bruteforce_config_a(oracle_mod):
    O = oracle_mod
    cfg = S.lidar_config("A")
    scene = S.scene_for("A")
    a = O.render_lidar(scene, cfg, mode="tiled")
    b = O.render_lidar(scene, cfg, mode="brute")
    for k in ("feat", "opacity", "depth_accum", "T_final", "n_contrib"):
        assert np.array_equal(a[k], b[k]), k
    assert (a["opacity"] > 0).mean() > 0.1


def test_tiled_equals_bruteforce_tiny_scenes(oracle_mod):
    O = oracle_mod
    for seed in range(100):
        cfg = S.lidar_config("tiny")
        if seed % 3 == 1:
            cfg.n_phi, cfg.max_rays_per_tile = 2, 64
        if seed % 3 == 2:
            cfg.cull_az_cells = 1600
        scene = S.scene_for("tiny", seed=seed)
        a = O.render_lidar(scene, cfg, mode="tiled", enable_cull=seed % 3)
        b = O.render_lidar(scene, cfg, mode="brute")
        for k in ("feat", "opacity", "depth_accum", "T_final", "n_contrib"):
            assert np.array_equal(a[k], b[k]), (seed, k)


def test_tiling_invariance_of_outputs(oracle_mod):
    """Tiling choice 'does not affect quality': outputs bit-identical across (N_phi, M)."""
    O = oracle_mod
    scene = S.scene_for("A")
    ref = None
    for n_phi, M in ((8, 32), (4, 64), (2, 256), (16, 16)):
        cfg = S.lidar_config("A")
        cfg.n_phi, cfg.max_rays_per_tile = n_phi, M
        out = O.render_lidar(scene, cfg)
        if ref is None:
            ref = out
        else:
            for k in ("feat", "opacity", "depth_accum", "T_final", "n_contrib"):
                assert np.array_equal(ref[k], out[k])


def test_bin_sets_and_order(oracle_mod):
    O = oracle_mod
    cfg = S.lidar_config("tiny")
    t = O.Tiling(cfg)
    scene = S.scene_for("tiny", seed=7)
    proj = O.project_lidar(scene, cfg)
    count, rect = O.cull_lidar(proj["valid"], proj["box"], t, False)
    keys, ids, ranges = O.bin_pairs(count, rect, proj["key"], t.n_tiles, t.n_theta)
    assert len(ids) == count.sum()
    kb = proj["key"].view(np.uint32)
    for tile in range(t.n_tiles):
        lo, hi = ranges[tile]
        lst = ids[lo:hi]
        expect = sorted([g for g in range(len(count)) if count[g] and
                         tile in {r * t.n_theta + (rect[g, 2] + c) % t.n_theta
                                  for r in range(rect[g, 0], rect[g, 1] + 1) for c in range(rect[g, 3])}],
                        key=lambda g: (kb[g], g))
        assert list(lst) == expect


def test_depth_key_is_float32_distance(oracle_mod):
    O = oracle_mod
    scene = S.scene_for("A")
    cfg = S.lidar_config("B")
    proj = O.project_lidar(scene, cfg)
    t0, t1 = cfg.pose_start["t"], cfg.pose_end["t"]
    om = (t0 + np.float32(0.5) * (t1 - t0)).astype(np.float32)
    d = (scene["means"] - om).astype(np.float32)
    key = np.sqrt(((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]).astype(np.float32))
    assert np.array_equal(key, proj["key"])


# ---------------------------------------------------------------- O6 camera
def test_camera_closed_forms(oracle_mod):
    O = oracle_mod
    cam = S.camera_config("D-small")
    cam.k = (0.0, 0.0, 0.0, 0.0, 0.0)  # equidistant fisheye: r = f theta
    p = np.array([1.0, 0, 0, 0, 0, 0, 0])
    for th in (0.0, 0.3, 1.0, 1.5):
        x = np.array([math.sin(th), 0.0, math.cos(th)]) * 5
        ok, uv = O.camera_point(x, cam, p, p, 0)
        assert ok and uv[0] == pytest.approx(cam.cx + cam.fx * th) and uv[1] == pytest.approx(cam.cy)
    pin = S.camera_config("pinhole-small")
    pin.k = (0.0,) * 5
    ok, uv = O.camera_point(np.array([1.0, -0.5, 4.0]), pin, p, p, 0)
    assert uv[0] == pytest.approx(pin.fx * 0.25 + pin.cx) and uv[1] == pytest.approx(pin.fy * -0.125 + pin.cy)
    # distorted models: unproject o project = identity
    for cfg in (S.camera_config("D-small"), S.camera_config("pinhole-small")):
        rng = np.random.default_rng(12)
        for _ in range(100):
            u, v = rng.uniform(0, cfg.width), rng.uniform(0, cfg.height)
            ok, d = O.camera_unproject(cfg, u, v)
            if not ok:
                continue
            ok2, uv = O.camera_point(d * 3.0, cfg, p, p, 0)
            assert ok2 and abs(uv[0] - u) < 1e-8 and abs(uv[1] - v) < 1e-8


@pytest.mark.parametrize("name", ["D", "D-small", "pinhole-small", "kb-random", "radtan-random"])
def test_camera_models_vs_opencv(oracle_mod, name):
    """O6 pinned to an independent implementation (A22): the oracle's KB fisheye
    and radtan projections equal OpenCV's cv2.fisheye.projectPoints / cv2.projectPoints, and
    its inverses equal cv2.fisheye.undistortPoints / cv2.undistortPointsIter, on >= 300
    random points inside the field of view (OpenCV's fisheye model is defined for z > 0)."""
    cv2 = pytest.importorskip("cv2")
    O = oracle_mod
    # a fixed seed per case (str hash() is salted per process)
    rng = np.random.default_rng({"D": 11, "D-small": 12, "pinhole-small": 13, "kb-random": 14,
                                 "radtan-random": 15}[name])
    if name == "kb-random":
        cam = S.camera_config("D-small")
        cam.k = tuple(rng.uniform(-0.01, 0.01, 4)) + (0.0,)
    elif name == "radtan-random":
        cam = S.camera_config("pinhole-small")
        cam.k = tuple(rng.uniform(-0.05, 0.05, 5))
    else:
        cam = S.camera_config(name)
    n = 300
    th_hi = min(cam.max_theta * 0.9, math.radians(89.0))
    if cam.model == 1:
        # the KB inverse is unique only where theta_d(theta) increases (A22): sample below the
        # first turning point of a random coefficient set
        tg = np.linspace(0.0, th_hi, 20001)
        k1, k2, k3, k4 = cam.k[:4]
        dth = 1 + 3 * k1 * tg**2 + 5 * k2 * tg**4 + 7 * k3 * tg**6 + 9 * k4 * tg**8
        if (dth <= 0).any():
            th_hi = 0.95 * tg[np.argmax(dth <= 0)]
    th = rng.uniform(0, th_hi, n)
    ph = rng.uniform(-math.pi, math.pi, n)
    r = rng.uniform(0.5, 50, n)
    X = np.stack([r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph), r * np.cos(th)], 1)
    f = lambda v: float(np.float32(v))  # noqa: E731  the interface's float32 camera parameters
    Km = np.array([[f(cam.fx), 0, f(cam.cx)], [0, f(cam.fy), f(cam.cy)], [0, 0, 1.0]])
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    ours = np.array([O.camera_point(x, cam, ident, ident, 0)[1][:2] for x in X])
    crit = (cv2.TERM_CRITERIA_COUNT | cv2.TERM_CRITERIA_EPS, 100, 1e-15)
    if cam.model == 1:
        D = np.array([f(v) for v in cam.k[:4]])
        ref, _ = cv2.fisheye.projectPoints(X.reshape(-1, 1, 3), np.zeros(3), np.zeros(3), Km, D)
        und = cv2.fisheye.undistortPoints(ours.reshape(-1, 1, 2), Km, D, criteria=crit).reshape(-1, 2)
    else:
        D = np.array([f(v) for v in cam.k])
        ref, _ = cv2.projectPoints(X.reshape(-1, 1, 3), np.zeros(3), np.zeros(3), Km, D)
        und = cv2.undistortPointsIter(ours.reshape(-1, 1, 2), Km, D, None, None, crit).reshape(-1, 2)
    assert np.abs(ours - ref.reshape(-1, 2)).max() < 1e-9  # pixels
    dirs = np.array([O.camera_unproject(cam, u, v)[1] for u, v in ours])
    rd = np.concatenate([und, np.ones((n, 1))], 1)
    rd /= np.linalg.norm(rd, axis=1, keepdims=True)
    # OpenCV's iterative undistortion does not always converge near 90 deg: compare where its
    # own answer reprojects onto the pixel
    if cam.model == 1:
        back, _ = cv2.fisheye.projectPoints(rd.reshape(-1, 1, 3), np.zeros(3), np.zeros(3), Km, D)
    else:
        back, _ = cv2.projectPoints(rd.reshape(-1, 1, 3), np.zeros(3), np.zeros(3), Km, D)
    conv = np.abs(back.reshape(-1, 2) - ours).max(1) < 1e-9
    assert conv.mean() > 0.9
    assert np.abs(dirs - rd)[conv].max() < 1e-12
    assert np.abs(dirs - X / np.linalg.norm(X, axis=1, keepdims=True)).max() < 1e-12


def test_camera_rolling_shutter_degenerate(oracle_mod):
    O = oracle_mod
    cam = S.camera_config("D-small")
    scene = S.scene_for("D", n=500)
    p = cam.pose_start
    a = O.project_camera(scene, cam, p, p, K=0)
    b = O.project_camera(scene, cam, p, p, K=3)
    assert np.array_equal(a["box"], b["box"], equal_nan=True) and np.array_equal(a["valid"], b["valid"])


def test_camera_ut_monte_carlo(oracle_mod):
    O = oracle_mod
    cam = S.camera_config("D-small")
    cam.rolling_shutter = 0
    p = S.pose([1, 0, 0, 0], [0, 0, 0])
    rng = np.random.default_rng(13)
    for mu, s in (((0.0, 0.0, 6.0), (0.2, 0.2, 0.2)), ((2.0, -1.0, 5.0), (0.3, 0.1, 0.2))):
        q = rng.normal(size=4)
        scene = {"means": np.array([mu], np.float32), "quats": np.array([q], np.float32),
                 "scales": np.array([s], np.float32), "opacity": np.array([0.9], np.float32),
                 "sh": np.zeros((1, 16, 3), np.float32)}
        proj = O.project_camera(scene, cam, p, p, K=0)
        Sig = O.covariance(q, np.asarray(s, np.float32).astype(np.float64))
        x = rng.multivariate_normal(np.asarray(mu, np.float32).astype(np.float64), Sig, 20000)
        uv = np.array([O.camera_point(xx, cam, pose_np(p), pose_np(p), 0)[1][:2] for xx in x])
        Cmc = np.cov(uv.T)
        c = proj["cov2d"][0]
        Cu = np.array([[c[0], c[1]], [c[1], c[2]]])
        assert np.linalg.norm(Cu - Cmc) / np.linalg.norm(Cmc) < 0.03


def pose_np(p):
    return np.r_[np.asarray(p["q"], np.float64), np.asarray(p["t"], np.float64)]


def test_camera_tiled_equals_bruteforce(oracle_mod):
    O = oracle_mod
    for name, seed in (("D-small", 1), ("pinhole-small", 2)):
        cam = S.camera_config(name)
        scene = S.corridor_scene(seed, 3000, x_range=(0.0, 40.0), kind="camera", ego=(1.5, 0, 1.6))
        a = O.render_camera(scene, cam, mode="tiled")
        b = O.render_camera(scene, cam, mode="brute")
        for k in ("feat", "opacity", "depth_accum", "T_final", "n_contrib"):
            assert np.array_equal(a[k], b[k]), (name, k)
        assert (a["opacity"] > 0.01).mean() > 0.05


# ------------------------------------------------------------------ beam divergence (App. C)
def test_divergence_cov_directions(oracle_mod):
    """Sigma_hat = Sigma + (theta r)^2 (I - d d^T): unchanged along the viewing
    direction, widened by exactly (theta r)^2 across it; for an isotropic particle the
    eigen-decomposition (numpy) is {a^2 along d, a^2 + (theta r)^2 twice}."""
    O = oracle_mod
    rng = np.random.default_rng(31)
    for _ in range(20):
        q, s = rng.normal(size=4), rng.uniform(0.02, 0.5, 3)
        Sig = O.covariance(q, s)
        mu, o = rng.uniform(-40, 40, 3), rng.uniform(-2, 2, 3)
        theta = rng.uniform(1e-4, 5e-3)
        Sh = O.divergence_cov(Sig, mu, o, theta)
        r = np.linalg.norm(mu - o)
        d = (mu - o) / r
        u = np.cross(d, rng.normal(size=3))
        u /= np.linalg.norm(u)
        assert np.allclose(Sh @ d, Sig @ d, atol=1e-12)
        assert abs(u @ Sh @ u - (u @ Sig @ u + (theta * r) ** 2)) < 1e-12
        assert np.allclose(Sh, Sh.T, atol=1e-15)
    a, theta = 0.07, 2e-3
    mu, o = np.array([30.0, -12.0, 1.0]), np.array([0.5, 0.2, 1.8])
    Sh = O.divergence_cov(a * a * np.eye(3), mu, o, theta)
    w, V = np.linalg.eigh(Sh)
    r = np.linalg.norm(mu - o)
    assert np.allclose(w, [a * a, a * a + (theta * r) ** 2, a * a + (theta * r) ** 2], rtol=1e-12)
    assert abs(abs(V[:, 0] @ (mu - o) / r) - 1.0) < 1e-12


def test_cholesky_and_lower_inverse(oracle_mod):
    """The oracle's textbook Cholesky equals numpy's; its triangular inverse inverts."""
    O = oracle_mod
    rng = np.random.default_rng(32)
    for _ in range(30):
        A = rng.normal(size=(3, 3))
        S = A @ A.T + 1e-3 * np.eye(3)
        L = O.cholesky3(S)
        assert np.allclose(L, np.linalg.cholesky(S), rtol=1e-12, atol=1e-14)
        assert np.allclose(O.lower_inverse3(L) @ L, np.eye(3), atol=1e-12)
    assert O.cholesky3(-np.eye(3)) is None


def test_divergence_response_closed_form_and_dense(oracle_mod):
    """Response with Sigma_hat (M_hat = chol(Sigma_hat)^-1): (i) a dense scan of the
    Mahalanobis distance along the ray with numpy's inv(Sigma_hat) gives the same minimum
    and argmin; (ii) for an isotropic particle seen from the sensor at angle beta off its
    centre, delta^2 = r^2 sin^2 b / (a^2 sin^2 b + (a^2 + (theta r)^2) cos^2 b) -- the
    beam footprint widens the particle across the beam only."""
    O = oracle_mod
    rng = np.random.default_rng(33)
    for _ in range(10):
        q, s = rng.normal(size=4), rng.uniform(0.05, 0.4, 3)
        mu, o = rng.uniform(-20, 20, 3), rng.uniform(-1, 1, 3)
        theta = 3e-3
        Sh = O.divergence_cov(O.covariance(q, s), mu, o, theta)
        M = O.lower_inverse3(O.cholesky3(Sh))
        d = (mu - o) + rng.normal(scale=0.3, size=3)
        d /= np.linalg.norm(d)
        tau, d2 = O.response(mu, M.reshape(-1), o, d)
        Si = np.linalg.inv(Sh)
        t = np.linspace(tau - 2.0, tau + 2.0, 200001)
        x = o[None, :] + t[:, None] * d[None, :] - mu[None, :]
        m = np.einsum("ni,ij,nj->n", x, Si, x)
        k = int(np.argmin(m))
        assert abs(m[k] - d2) < 1e-6 * max(1.0, d2) and abs(t[k] - tau) < 2e-5
    a, theta, r = 0.05, 2e-3, 40.0
    mu, o = np.array([r, 0.0, 0.0]), np.zeros(3)
    Sh = O.divergence_cov(a * a * np.eye(3), mu, o, theta)
    M = O.lower_inverse3(O.cholesky3(Sh))
    b2 = a * a + (theta * r) ** 2
    for beta in (0.0, 1e-4, 1e-3, 4e-3, 2e-2):
        d = np.array([np.cos(beta), np.sin(beta), 0.0])
        _, d2 = O.response(mu, M.reshape(-1), o, d)
        ref = r * r * np.sin(beta) ** 2 / (a * a * np.sin(beta) ** 2 + b2 * np.cos(beta) ** 2)
        assert abs(d2 - ref) <= 1e-9 * max(1.0, ref), (beta, d2, ref)


def test_ut_affine_exact_with_cholesky_root(oracle_mod):
    """UT with the Cholesky root of Sigma_hat through an affine sensor is exact:
    mean A mu + b, covariance A Sigma_hat A^T (the UT moments written out here)."""
    O = oracle_mod
    rng = np.random.default_rng(34)
    for ut in ((1.0, 2.0, 0.0), (0.6, 2.0, 0.5)):
        Sh = O.divergence_cov(O.covariance(rng.normal(size=4), rng.uniform(0.05, 0.5, 3)),
                              rng.uniform(-10, 10, 3), np.zeros(3), 4e-3)
        mu = rng.uniform(-10, 10, 3)
        pts, wm, wc = O.sigma_points_sqrt(mu, O.cholesky3(Sh), ut)
        A, b = rng.normal(size=(2, 3)), rng.normal(size=2)
        y = pts @ A.T + b
        mean = wm @ y
        cov = (wc[:, None, None] * np.einsum("ni,nj->nij", y - mean, y - mean)).sum(0)
        assert np.allclose(mean, A @ mu + b, atol=1e-9)
        assert np.allclose(cov, A @ Sh @ A.T, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("theta", [1.5e-3, 5e-3])
def test_divergence_tiled_equals_bruteforce_and_widens(oracle_mod, theta):
    """With the filter on, tiling and culling stay exact accelerations (tiled = brute force
    on tiny scenes, A12); and since Sigma_hat - Sigma is positive semi-definite, every
    (ray, particle) Mahalanobis distance can only shrink: delta_hat^2 <= delta^2."""
    O = oracle_mod
    for seed in range(6):
        cfg = S.lidar_config("tiny")
        scene = S.scene_for("tiny", seed=seed)
        cfg.beam_divergence = theta
        tiled = O.render_lidar(scene, cfg)
        brute = O.render_lidar(scene, cfg, mode="brute")
        for k in ("feat", "opacity", "depth_accum", "T_final"):
            assert np.array_equal(tiled[k], brute[k]), k
    rng = np.random.default_rng(35)
    for _ in range(200):
        q, s = rng.normal(size=4), rng.uniform(0.02, 0.5, 3)
        mu, o = rng.uniform(-30, 30, 3), rng.uniform(-1, 1, 3)
        Sig = O.covariance(q, s)
        M = O.lower_inverse3(O.cholesky3(Sig))
        Mh = O.lower_inverse3(O.cholesky3(O.divergence_cov(Sig, mu, o, theta)))
        d = (mu - o) + rng.normal(scale=2.0, size=3)
        d /= np.linalg.norm(d)
        assert O.response(mu, Mh.reshape(-1), o, d)[1] <= O.response(mu, M.reshape(-1), o, d)[1] * (1 + 1e-9) + 1e-12


# ------------------------------------------------------------------ camera Eq. 2
def _dirs(lon, colat):
    return np.stack([np.sin(colat) * np.cos(lon), np.sin(colat) * np.sin(lon), np.cos(colat)], -1)


def test_compose_identity_and_constant_background(oracle_mod):
    """Eq. 2 with A = identity: c = omega c_f + (1 - omega) c_b, where omega c_f is the
    renderer's Eq. 1 sum (A28); a constant environment gives c_b = that constant for every
    direction; no map, no grid: c = the Eq. 1 sum."""
    O = oracle_mod
    cam = S.camera_config("D-small")
    rng = np.random.default_rng(41)
    n = cam.width * cam.height
    od = np.zeros((n, 6))
    od[:, 3:] = rng.normal(size=(n, 3))
    cf, om = rng.uniform(0, 1, (n, 3)), rng.uniform(0, 1, n)
    k = np.array([0.2, 0.5, 0.9], np.float32)
    env = np.broadcast_to(k, (7, 13, 3)).copy()
    ident = np.zeros((3, 4, 5, 12), np.float32)
    ident[..., 0] = ident[..., 5] = ident[..., 10] = 1.0
    out = O.compose_camera(cam, od, cf, om, env, ident)
    assert np.allclose(out, cf + (1 - om[:, None]) * k.astype(np.float64), atol=1e-6)
    assert np.allclose(O.compose_camera(cam, od, cf, om), cf, atol=1e-15)


def test_compose_env_bilinear(oracle_mod):
    """The equirectangular lookup returns a texel's value at its centre direction, the mean of
    two neighbours halfway between them, and wraps across longitude +-pi."""
    O = oracle_mod
    cam = S.camera_config("D-small")
    He, We = 6, 10
    rng = np.random.default_rng(42)
    env = rng.uniform(0, 1, (He, We, 3)).astype(np.float32)
    i, j = 2, 3
    lon = (j + 0.5) / We * 2 * np.pi - np.pi
    colat = (i + 0.5) / He * np.pi
    lon_half = (j + 1.0) / We * 2 * np.pi - np.pi
    lon_wrap = np.pi - 1e-12  # between the last column and the first (u = We - 0.5 ~ -0.5 wrapped)
    d = np.array([_dirs(lon, colat), _dirs(lon_half, colat), _dirs(lon_wrap, colat)])
    n = cam.width * cam.height
    od = np.zeros((n, 6))
    od[:3, 3:] = d
    out = O.compose_camera(cam, od, np.zeros((n, 3)), np.zeros(n), env, None)
    assert np.allclose(out[0], env[i, j], atol=1e-9)
    assert np.allclose(out[1], 0.5 * (env[i, j] + env[i, j + 1]), atol=1e-9)
    assert np.allclose(out[2], 0.5 * (env[i, We - 1] + env[i, 0]), atol=1e-6)


def test_compose_grid_trilinear_exact_for_affine_fields(oracle_mod):
    """A bilateral grid whose 12 coefficients are an affine function of the cell-centre
    coordinates reproduces that function exactly inside the grid (trilinear interpolation
    is exact for affine fields); checked against the field evaluated directly."""
    O = oracle_mod
    cam = S.camera_config("D-small")
    W, H = cam.width, cam.height
    gd, gh, gw = 4, 5, 6
    rng = np.random.default_rng(43)
    Acoef = rng.normal(scale=0.1, size=(12, 3))
    b = rng.normal(scale=0.1, size=12)
    zc, yc, xc = np.meshgrid((np.arange(gd) + 0.5) / gd, (np.arange(gh) + 0.5) / gh, (np.arange(gw) + 0.5) / gw,
                             indexing="ij")
    grid = (np.stack([xc, yc, zc], -1) @ Acoef.T + b).astype(np.float64)
    n = W * H
    cf = rng.uniform(0.2, 0.8, (n, 3))
    om = np.ones(n)
    out = O.compose_camera(cam, np.zeros((n, 6)), cf, om, None, grid.astype(np.float32))
    px, py = (np.arange(n) % W + 0.5) / W, (np.arange(n) // W + 0.5) / H
    lum = np.clip(0.299 * cf[:, 0] + 0.587 * cf[:, 1] + 0.114 * cf[:, 2], 0, 1)
    inside = (px > 0.5 / gw) & (px < 1 - 0.5 / gw) & (py > 0.5 / gh) & (py < 1 - 0.5 / gh) & \
             (lum > 0.5 / gd) & (lum < 1 - 0.5 / gd)
    M = np.stack([px, py, lum], -1) @ Acoef.T + b  # the field itself (float64)
    M = M.reshape(n, 3, 4)
    ref = np.einsum("nij,nj->ni", M[:, :, :3], cf) + M[:, :, 3]
    assert inside.mean() > 0.3
    assert np.abs(out - ref)[inside].max() < 1e-6  # (grid stored as float32)


# ------------------------------------------------------------------ scene graph (O0)
def test_actors_to_world_vs_scipy(oracle_mod):
    """O0: mu_w = R_a mu + t_a (scipy Rotation, double) rounded to float32 (<= 1 ulp);
    Sigma_w = R_a Sigma R_a^T (scipy); static particles bit-unchanged; an out-of-range id
    gives a zero quaternion (invalid particle)."""
    O = oracle_mod
    base = S.corridor_scene(5, 300, x_range=(0.0, 40.0))
    sc = S.with_actors(base, 6, n_actors=5, per_actor=60)
    sc["actor_id"][:3] = [7, -2, 5]  # out of range
    w = O.actors_to_world(sc)
    ids = sc["actor_id"]
    st = ids == -1
    assert np.array_equal(w["means"][st].view(np.uint32), sc["means"][st].view(np.uint32))
    assert np.array_equal(w["quats"][st].view(np.uint32), sc["quats"][st].view(np.uint32))
    assert np.all(w["quats"][:3] == 0)
    P = sc["actor_pose"].astype(np.float64)
    for i in np.nonzero((ids >= 0) & (ids < 5))[0]:
        Ra = Rotation.from_quat(P[ids[i], [1, 2, 3, 0]]).as_matrix()
        ref = Ra @ sc["means"][i].astype(np.float64) + P[ids[i], 4:]
        assert np.all(np.abs(w["means"][i] - ref) <= np.spacing(np.abs(ref).astype(np.float32)))
        ql = sc["quats"][i].astype(np.float64)
        Rl = Rotation.from_quat(ql[[1, 2, 3, 0]]).as_matrix()
        Sl = Rl @ np.diag(sc["scales"][i].astype(np.float64) ** 2) @ Rl.T
        Sw = O.covariance(w["quats"][i].astype(np.float64), sc["scales"][i].astype(np.float64))
        assert np.allclose(Sw, Ra @ Sl @ Ra.T, rtol=0, atol=1e-6 * np.abs(Sl).max())
    pr = O.project_lidar(sc, S.lidar_config("A"))
    assert np.all(pr["valid"][:3] == 0)


def test_actor_rigid_invariance_lidar(oracle_mod):
    """Moving the whole scene as one object by P and the sensor by P too (sensor pose
    P o X) leaves the scan unchanged (rigid invariance of Eq. 3 / the response); compared
    with the local scene scanned from X.  Differences come only from rounding the world
    means to float32 and from rays near a decision threshold (flagged)."""
    O = oracle_mod
    cfg = S.lidar_config("tiny")
    scene = S.scene_for("tiny", seed=31, n=300)
    qP = np.array([np.cos(0.35), 0.05, -0.03, np.sin(0.35)])
    qP /= np.linalg.norm(qP)
    tP = np.array([12.0, -4.0, 0.5])
    sc = dict(scene)
    sc["actor_id"] = np.zeros(scene["means"].shape[0], np.int32)
    sc["actor_pose"] = np.concatenate([qP, tP])[None].astype(np.float32)
    P32 = sc["actor_pose"][0].astype(np.float64)
    RP = Rotation.from_quat(P32[[1, 2, 3, 0]])
    def moved(X):  # P o X
        RX = Rotation.from_quat(np.asarray(X["q"], np.float64)[[1, 2, 3, 0]])
        return S.pose((RP * RX).as_quat()[[3, 0, 1, 2]], RP.apply(np.asarray(X["t"], np.float64)) + P32[4:])

    LIDAR_EPS_PIN = {"a": 3e-6, "b": 3e-6, "alpha": 1e-5, "T_rel": 1e-3, "tau": 1e-3, "impact": 5e-5}
    ref = O.render_lidar(scene, cfg, flag_eps=LIDAR_EPS_PIN)
    got = O.render_lidar(sc, cfg, pose0=moved(cfg.pose_start), pose1=moved(cfg.pose_end), flag_eps=LIDAR_EPS_PIN)
    ok = (ref["flag"] == 0) & (got["flag"] == 0)
    assert ok.mean() > 0.97
    assert (ref["opacity"] > 0.1).mean() > 0.05
    assert np.abs(got["opacity"] - ref["opacity"])[ok].max() < 2e-5
    hit = ok & (ref["opacity"] > 0.5)
    assert np.abs(got["depth"] - ref["depth"])[hit].max() < 1e-4


# ------------------------------------------------------------------ per-ray SH (Eq. 1 literally, A30)
def test_per_ray_sh_closed_forms(oracle_mod):
    """Per-ray SH (zeta = sum_i SH_i(d) alpha_i T_i, d the ray direction): (1) degree 0: the
    same as per-particle features (Y_00 is constant); (2) every particle with the same
    coefficients c: zeta(r) = omega(r) SH_c(d_r) exactly (sh_eval is pinned against scipy
    above), whereas per-particle features are not -- they see each particle's own view
    direction."""
    O = oracle_mod
    cfg = S.lidar_config("tiny")
    scene = S.scene_for("tiny", seed=17, n=400)
    s0 = dict(scene)
    s0["sh"] = np.ascontiguousarray(scene["sh"][:, :1])
    a = O.render_lidar(s0, cfg)
    b = O.render_lidar(s0, cfg, per_ray_sh=True)
    assert np.abs(a["feat"] - b["feat"]).max() < 1e-13
    assert np.array_equal(a["opacity"], b["opacity"])
    rng = np.random.default_rng(18)
    c = rng.normal(size=(16, 3))
    s1 = dict(scene)
    s1["sh"] = np.ascontiguousarray(np.broadcast_to(c.astype(np.float32), scene["sh"].shape))
    pr = O.render_lidar(s1, cfg, per_ray_sh=True)
    pp = O.render_lidar(s1, cfg)
    od = pr["ray_od"]
    hit = pr["opacity"] > 0.05
    assert hit.mean() > 0.05
    for r in np.nonzero(hit)[0][:200]:
        d = od[r, 3:] / np.linalg.norm(od[r, 3:])
        ref = pr["opacity"][r] * O.sh_eval(c.astype(np.float32).astype(np.float64), d)
        assert np.allclose(pr["feat"][r], ref, rtol=0, atol=1e-12)
    assert np.abs(pp["feat"] - pr["feat"])[hit].max() > 1e-3  # the two readings differ


# ------------------------------------------------------------------ backward (O15, O16; A31)
def _bwd_setup(O, seed=3, n=120, deg0=True):
    cfg = S.lidar_config("tiny")
    sc = S.scene_for("tiny", seed=seed, n=n)
    if deg0:  # constant features: the SH view direction carries no gradient (A31)
        sc["sh"] = np.ascontiguousarray(sc["sh"][:, :1])
    fwd = O.render_lidar(sc, cfg)
    R = fwd["opacity"].shape[0]
    rng = np.random.default_rng(seed + 100)
    g = {"zeta": rng.normal(size=(R, 3)), "opacity": rng.normal(size=R), "depth_accum": rng.normal(size=R) * 0.1,
         "depth": rng.normal(size=R) * 0.1, "intensity": rng.normal(size=R), "raydrop": rng.normal(size=R)}
    return cfg, sc, g


def _loss(O, sc, cfg, g):
    f = O.render_lidar(sc, cfg)
    return (np.sum(g["zeta"] * f["feat"]) + np.sum(g["opacity"] * f["opacity"]) +
            np.sum(g["depth_accum"] * f["depth_accum"]) + np.sum(g["depth"] * f["depth"]) +
            np.sum(g["intensity"] * f["intensity"]) + np.sum(g["raydrop"] * f["raydrop"]))


def test_backward_vs_finite_differences(oracle_mod):
    """O15/O16 against central differences of the oracle's own forward (a different
    computation: the derivative is fixed by the forward map).  The particles with the
    largest gradients are perturbed in every parameter (mean, quaternion, scale, opacity);
    the step is small enough that no membership / skip / termination decision flips for
    almost all of them."""
    O = oracle_mod
    cfg, sc, g = _bwd_setup(O)
    b = O.backward_lidar(sc, cfg, g)
    top = np.argsort(-np.abs(b["opacity"]))[:6]
    checked = bad = 0
    for i in top:
        for key, h, dims in (("means", 2e-4, 3), ("quats", 2e-4, 4), ("scales", 1e-4, 3), ("opacity", 1e-4, 1)):
            for c in range(dims):
                vals = []
                deltas = []
                for sgn in (1, -1):
                    s2 = {k: v.copy() for k, v in sc.items()}
                    arr = s2[key].reshape(sc["means"].shape[0], -1)
                    x0 = np.float32(arr[i, c])
                    arr[i, c] = np.float32(x0 + sgn * h * max(1.0, abs(float(x0))))
                    deltas.append(float(arr[i, c]) - float(x0))
                    vals.append(_loss(O, s2, cfg, g))
                fd = (vals[0] - vals[1]) / (deltas[0] - deltas[1])
                an = b[key].reshape(sc["means"].shape[0], -1)[i, c]
                checked += 1
                if abs(fd - an) > 2e-3 * max(1.0, abs(an)):
                    bad += 1
                    print("mismatch", i, key, c, fd, an)
    assert checked == 6 * 11
    assert bad <= 2, bad  # a decision flip inside the stencil is possible but rare


def test_backward_sh_exact_linearity(oracle_mod):
    """zeta is linear in the SH coefficients: L(c + e_k) - L(c) = dL/dc_k exactly (up to
    rounding) for a loss linear in zeta, on the particles with the largest SH gradients."""
    O = oracle_mod
    cfg, sc, g = _bwd_setup(O, seed=4, deg0=False)
    g["raydrop"][:] = 0.0  # the sigmoid of the ray-drop decode is not linear in zeta
    b = O.backward_lidar(sc, cfg, g)
    L0 = _loss(O, sc, cfg, g)
    top = np.argsort(-np.abs(b["sh"]).sum((1, 2)))[:3]
    for i in top:
        for k in (0, 1, 5, 15):
            for c in range(3):
                s2 = {kk: v.copy() for kk, v in sc.items()}
                s2["sh"][i, k, c] += np.float32(0.5)
                d = float(s2["sh"][i, k, c]) - float(sc["sh"][i, k, c])
                assert abs((_loss(O, s2, cfg, g) - L0) / d - b["sh"][i, k, c]) < 1e-9 * max(1, abs(b["sh"][i, k, c]))


def test_backward_transmittance_identity(oracle_mod):
    """Euler-type identity: scaling every opacity sigma -> (1 + e) sigma changes
    sum_r omega_r = sum_r (1 - T_final,r) at rate sum_i sigma_i dL/dsigma_i (G_omega = 1);
    the rate is taken from T_final (omega = 1 - T, Eq. 1), not from the backward."""
    O = oracle_mod
    cfg = S.lidar_config("tiny")
    sc = S.scene_for("tiny", seed=9, n=150)
    sc["opacity"] = (sc["opacity"] * 0.5).astype(np.float32)  # no clamping at alpha_max
    fwd = O.render_lidar(sc, cfg)
    R = fwd["opacity"].shape[0]
    b = O.backward_lidar(sc, cfg, {"opacity": np.ones(R)})
    e = 1e-4
    s2 = dict(sc)
    s2["opacity"] = (sc["opacity"].astype(np.float64) * (1 + e)).astype(np.float32)
    s3 = dict(sc)
    s3["opacity"] = (sc["opacity"].astype(np.float64) * (1 - e)).astype(np.float32)
    f2, f3 = O.render_lidar(s2, cfg), O.render_lidar(s3, cfg)
    fd = (np.sum(1 - f2["T_final"]) - np.sum(1 - f3["T_final"])) / (2 * e)
    an = np.sum(sc["opacity"].astype(np.float64) * b["opacity"])
    assert np.allclose(f2["opacity"], 1 - f2["T_final"], atol=1e-12)  # omega = 1 - T (Eq. 1)
    assert abs(fd - an) < 1e-3 * max(1.0, abs(an)), (fd, an)


def test_backward_camera_vs_finite_differences(oracle_mod):
    """O15/O16 on the camera path (KB fisheye, rolling shutter) against central differences
    of the oracle's camera forward: loss = sum of random weights x (rgb, omega, D, depth)."""
    O = oracle_mod
    cam = S.camera_config("D-small")
    cam.width, cam.height, cam.cx, cam.cy = 96, 64, 48.0, 32.0
    sc = S.corridor_scene(12, 2500, x_range=(3.0, 25.0), kind="camera", ego=(1.5, 0.0, 1.6))
    sc["sh"] = np.ascontiguousarray(sc["sh"][:, :1])  # constant colour: no view-direction term (A31)
    R = cam.width * cam.height
    rng = np.random.default_rng(13)
    g = {"rgb": rng.normal(size=(R, 3)), "opacity": rng.normal(size=R), "depth_accum": 0.05 * rng.normal(size=R),
         "depth": 0.05 * rng.normal(size=R)}

    def loss(s):
        f = O.render_camera(s, cam)
        return (np.sum(g["rgb"] * f["feat"]) + np.sum(g["opacity"] * f["opacity"]) +
                np.sum(g["depth_accum"] * f["depth_accum"]) + np.sum(g["depth"] * f["depth"]))

    b = O.backward_camera(sc, cam, g)
    assert (b["fwd"]["opacity"] > 0.1).mean() > 0.05
    top = np.argsort(-np.abs(b["opacity"]))[:4]
    checked = bad = 0
    for i in top:
        for key, h, dims in (("means", 2e-4, 3), ("quats", 2e-4, 4), ("scales", 1e-4, 3), ("opacity", 1e-4, 1)):
            for c in range(dims):
                vals, deltas = [], []
                for sgn in (1, -1):
                    s2 = {k: v.copy() for k, v in sc.items()}
                    arr = s2[key].reshape(sc["means"].shape[0], -1)
                    x0 = np.float32(arr[i, c])
                    arr[i, c] = np.float32(x0 + sgn * h * max(1.0, abs(float(x0))))
                    deltas.append(float(arr[i, c]) - float(x0))
                    vals.append(loss(s2))
                fd = (vals[0] - vals[1]) / (deltas[0] - deltas[1])
                an = b[key].reshape(sc["means"].shape[0], -1)[i, c]
                checked += 1
                if abs(fd - an) > 2e-3 * max(1.0, abs(an)):
                    bad += 1
                    print("mismatch", i, key, c, fd, an)
    assert checked == 4 * 11 and bad <= 2, bad


def test_backward_scene_graph_vs_finite_differences(oracle_mod):
    """O16 through the scene graph (A29, A31): gradients of object-frame particle
    parameters and of the object poses (q_a, t_a) against central differences of the
    oracle's forward."""
    O = oracle_mod
    cfg = S.lidar_config("tiny")
    base = S.scene_for("tiny", seed=21, n=80)
    sc = S.with_actors(base, 22, n_actors=2, per_actor=60, x_range=(3.0, 6.0))
    sc["actor_pose"][:, 5] = np.array([2.5, -3.0], np.float32)  # near the sensor, inside the beams
    sc["actor_pose"][:, 6] = 0.6
    sc["sh"] = np.ascontiguousarray(sc["sh"][:, :1])
    fwd = O.render_lidar(sc, cfg)
    R = fwd["opacity"].shape[0]
    rng = np.random.default_rng(23)
    g = {"zeta": rng.normal(size=(R, 3)), "opacity": rng.normal(size=R), "depth_accum": 0.1 * rng.normal(size=R),
         "depth": 0.1 * rng.normal(size=R), "intensity": rng.normal(size=R), "raydrop": rng.normal(size=R)}
    b = O.backward_lidar(sc, cfg, g)
    ids = sc["actor_id"]
    assert np.abs(b["actor_pose"]).max() > 0

    def fd(key, idx, h):
        vals, deltas = [], []
        for sgn in (1, -1):
            s2 = {k: v.copy() for k, v in sc.items()}
            arr = s2[key].reshape(s2[key].shape[0], -1)
            x0 = np.float32(arr[idx])
            arr[idx] = np.float32(x0 + sgn * h * max(1.0, abs(float(x0))))
            deltas.append(float(arr[idx]) - float(x0))
            vals.append(_loss(O, s2, cfg, g))
        return (vals[0] - vals[1]) / (deltas[0] - deltas[1])

    checked = bad = 0
    for a in range(2):
        for c in range(7):
            an = b["actor_pose"][a, c]
            num = fd("actor_pose", (a, c), 1e-4)
            checked += 1
            # a pose step moves every object mean, and the forward rounds each world mean to
            # float32 (A29): ~2.4e-7 m of quantisation per particle against a 1e-4 x 3 m step
            # puts ~1e-2 of noise on the difference quotient (measured agreement 1e-4 .. 3e-2)
            if abs(num - an) > 2e-3 * abs(an) + 0.05:
                bad += 1
                print("mismatch pose", a, c, num, an)
    top = [i for i in np.argsort(-np.abs(b["opacity"])) if ids[i] >= 0][:3]
    for i in top:
        for key, h, dims in (("means", 2e-4, 3), ("quats", 2e-4, 4), ("scales", 1e-4, 3)):
            for c in range(dims):
                an = b[key].reshape(len(ids), -1)[i, c]
                num = fd(key, (i, c), h)
                checked += 1
                if abs(num - an) > 2e-3 * max(1.0, abs(an)):
                    bad += 1
                    print("mismatch", i, key, c, num, an)
    assert checked == 14 + 3 * 10 and bad <= 2, bad


def test_backward_per_ray_sh_vs_finite_differences(oracle_mod):
    """Per-ray SH (A30) backward: the features SH_i(d) do not depend on the particle's
    position, so central differences of the forward check every parameter at full SH
    degree 3; the SH gradient (per (ray, particle) basis) is exact by linearity."""
    O = oracle_mod
    cfg = S.lidar_config("tiny")
    sc = S.scene_for("tiny", seed=33, n=120)
    fwd = O.render_lidar(sc, cfg, per_ray_sh=True)
    R = fwd["opacity"].shape[0]
    rng = np.random.default_rng(34)
    g = {"zeta": rng.normal(size=(R, 3)), "opacity": rng.normal(size=R), "depth_accum": 0.1 * rng.normal(size=R),
         "depth": 0.1 * rng.normal(size=R), "intensity": rng.normal(size=R), "raydrop": np.zeros(R)}
    b = O.backward_lidar(sc, cfg, g, per_ray_sh=True)

    def loss(s):
        f = O.render_lidar(s, cfg, per_ray_sh=True)
        return (np.sum(g["zeta"] * f["feat"]) + np.sum(g["opacity"] * f["opacity"]) +
                np.sum(g["depth_accum"] * f["depth_accum"]) + np.sum(g["depth"] * f["depth"]) +
                np.sum(g["intensity"] * f["intensity"]))

    L0 = loss(sc)
    top = np.argsort(-np.abs(b["sh"]).sum((1, 2)))[:2]
    for i in top:
        for k in (0, 3, 9, 15):
            s2 = {kk: v.copy() for kk, v in sc.items()}
            s2["sh"][i, k, 1] += np.float32(0.5)
            d = float(s2["sh"][i, k, 1]) - float(sc["sh"][i, k, 1])
            assert abs((loss(s2) - L0) / d - b["sh"][i, k, 1]) < 1e-9 * max(1, abs(b["sh"][i, k, 1]))
    checked = bad = 0
    # small steps: the top particle sits 0.7 m from the sensor, where a 2e-4 step already
    # flips a membership decision (the derivative itself matches to 1e-9 at 5e-5)
    for i in np.argsort(-np.abs(b["opacity"]))[:3]:
        for key, h, dims in (("means", 5e-5, 3), ("scales", 3e-5, 3), ("opacity", 1e-4, 1)):
            for c in range(dims):
                vals, deltas = [], []
                for sgn in (1, -1):
                    s2 = {kk: v.copy() for kk, v in sc.items()}
                    arr = s2[key].reshape(sc["means"].shape[0], -1)
                    x0 = np.float32(arr[i, c])
                    arr[i, c] = np.float32(x0 + sgn * h * max(1.0, abs(float(x0))))
                    deltas.append(float(arr[i, c]) - float(x0))
                    vals.append(loss(s2))
                num = (vals[0] - vals[1]) / (deltas[0] - deltas[1])
                an = b[key].reshape(sc["means"].shape[0], -1)[i, c]
                checked += 1
                if abs(num - an) > 2e-3 * max(1.0, abs(an)):
                    bad += 1
                    print("mismatch", i, key, c, num, an)
    assert checked == 21 and bad <= 1, bad


def test_backward_beam_divergence_vs_finite_differences(oracle_mod):
    """App. C backward (A27, A31): M_hat = chol(Sigma_hat)^-1 differentiated through the
    Cholesky factor (Sigma_bar = sym(M^T Phi(L^T Lbar) M)) and Sigma_hat's dependence on the
    view vector; central differences of the forward on a static-pose sensor (the sensor
    position does not move with the mean's firing time)."""
    O = oracle_mod
    cfg = S.lidar_config("A")
    cfg.beam_divergence = 5e-3
    sc = S.scene_for("A", seed=41, n=400)
    sc["sh"] = np.ascontiguousarray(sc["sh"][:, :1])
    fwd = O.render_lidar(sc, cfg)
    R = fwd["opacity"].shape[0]
    rng = np.random.default_rng(42)
    g = {"zeta": rng.normal(size=(R, 3)), "opacity": rng.normal(size=R), "depth_accum": 0.1 * rng.normal(size=R),
         "depth": 0.1 * rng.normal(size=R), "intensity": rng.normal(size=R), "raydrop": rng.normal(size=R)}
    b = O.backward_lidar(sc, cfg, g)
    checked = bad = 0
    for i in np.argsort(-np.abs(b["opacity"]))[:4]:
        for key, h, dims in (("means", 1e-4, 3), ("quats", 1e-4, 4), ("scales", 5e-5, 3)):
            for c in range(dims):
                vals, deltas = [], []
                for sgn in (1, -1):
                    s2 = {k: v.copy() for k, v in sc.items()}
                    arr = s2[key].reshape(sc["means"].shape[0], -1)
                    x0 = np.float32(arr[i, c])
                    arr[i, c] = np.float32(x0 + sgn * h * max(1.0, abs(float(x0))))
                    deltas.append(float(arr[i, c]) - float(x0))
                    vals.append(_loss(O, s2, cfg, g))
                num = (vals[0] - vals[1]) / (deltas[0] - deltas[1])
                an = b[key].reshape(sc["means"].shape[0], -1)[i, c]
                checked += 1
                if abs(num - an) > 2e-3 * max(1.0, abs(an)):
                    bad += 1
                    print("mismatch", i, key, c, num, an)
    assert checked == 40 and bad <= 2, bad
