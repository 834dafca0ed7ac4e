"""Seeded synthetic inputs (scenes, sensors, poses) shared by the CUDA path and the oracle.

This module holds NONE of the method's arithmetic: it only draws numbers with
``numpy.random.default_rng(seed)`` and lays them out in the C-ABI input format
(float32, row-major).  Recipes follow SURVEY.md §8(d) / DESIGN.md §5 and the paper's
workload description:

* LiDAR Gaussians come from voxelised LiDAR at 0.1 m -> surface-like, thin
  Gaussians on ground / facades / objects; opacities pushed to binary by the entropy
  loss -> bimodal opacity.
* Camera Gaussians are unconstrained volumetric particles.
* Driving scenes (Waymo / PandaSet) -> a straight road corridor.

Poses are (q[w,x,y,z], t[3]) float32, sensor -> world.  The rotation quaternion for a
yaw angle is written in closed form here only to *describe* an input pose.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

Y00 = 0.28209479177387814  # real-SH DC constant, used only to scale drawn DC values

# ------------------------------------------------------------------------------------
# poses
# ------------------------------------------------------------------------------------


def yaw_quat(yaw: float, base: np.ndarray | None = None) -> np.ndarray:
    """Quaternion (w,x,y,z) of a rotation by ``yaw`` about world z, optionally
    composed with ``base`` (q_yaw * base)."""
    qz = np.array([math.cos(yaw / 2), 0.0, 0.0, math.sin(yaw / 2)])
    if base is None:
        return qz.astype(np.float32)
    w1, x1, y1, z1 = qz
    w2, x2, y2, z2 = base
    return np.array([
        w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
        w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
        w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
        w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2,
    ], dtype=np.float32)


def pose(q, t) -> dict:
    return {"q": np.asarray(q, np.float32).reshape(4), "t": np.asarray(t, np.float32).reshape(3)}


# OpenCV camera (x right, y down, z forward) looking along world +x, z up:
# columns of R_cam->world are x_cam=(0,-1,0), y_cam=(0,0,-1), z_cam=(1,0,0)  -> q below.
CAM_FORWARD_Q = np.array([0.5, -0.5, 0.5, -0.5], dtype=np.float32)

# ------------------------------------------------------------------------------------
# sensors
# ------------------------------------------------------------------------------------


def pandar64_beams() -> np.ndarray:
    """Pandar64-like irregular beam table (deg -> rad), SURVEY §8(d) config B."""
    top = [15.0, 11.0, 8.0, 5.0, 3.0]
    mid = list(np.linspace(2.0, -6.0, 49))
    bot = [-7.0, -8.0, -9.0, -10.0, -11.0, -12.0, -13.0, -14.0, -19.0, -25.0]
    return np.radians(np.array(top + mid + bot, dtype=np.float64)).astype(np.float32)


def waymo_top_beams() -> np.ndarray:
    """Waymo-top-like: omega_b = 2.4 deg - 20 deg (b/63)^1.5 (dense near the horizon)."""
    b = np.arange(64, dtype=np.float64)
    return np.radians(2.4 - 20.0 * (b / 63.0) ** 1.5).astype(np.float32)


def uniform_beams(n: int, lo_deg: float, hi_deg: float) -> np.ndarray:
    return np.radians(np.linspace(lo_deg, hi_deg, n)).astype(np.float32)


@dataclass
class LidarConfig:
    name: str
    beams: np.ndarray
    n_azimuth: int
    n_phi: int = 16
    max_rays_per_tile: int = 32
    hist_bins: int = 400
    cull_az_cells: int = 1600
    cull_rows_per_tile: int = 8
    azimuth_start: float = float(np.float32(-math.pi))
    spin_direction: int = 1
    min_range: float = 0.1
    rs_iterations: int = 1
    beam_divergence: float = 0.0  # theta_div (rad), App. C filter; 0 = off (A24); SPEC suggests 1.5e-3
    pose_start: dict = field(default_factory=lambda: pose([1, 0, 0, 0], [0, 0, 1.8]))
    pose_end: dict = field(default_factory=lambda: pose([1, 0, 0, 0], [0, 0, 1.8]))

    @property
    def n_rays(self) -> int:
        return int(self.beams.shape[0]) * self.n_azimuth


@dataclass
class CameraConfig:
    name: str
    model: int  # 0 pinhole+radtan, 1 KB fisheye
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    k: tuple
    rolling_shutter: int = 1
    near: float = 0.05
    max_theta: float = math.radians(100.0)
    tile_px: int = 16
    rs_iterations: int = 1
    pose_start: dict = field(default_factory=lambda: pose(CAM_FORWARD_Q, [1.5, 0, 1.6]))
    pose_end: dict = field(default_factory=lambda: pose(CAM_FORWARD_Q, [1.5, 0, 1.6]))

    @property
    def n_pixels(self) -> int:
        return self.width * self.height


def lidar_config(name: str) -> LidarConfig:
    """BASELINE.json configs: 'A' 32x512 static, 'B' Pandar64 64x1800 rolling shutter,
    'C' Waymo-top 64x2650; 'tiny' 8x64 for brute-force pins."""
    if name == "A":
        return LidarConfig("A", uniform_beams(32, -30.0, 10.0), 512, n_phi=8, rs_iterations=1)
    if name == "B":
        return LidarConfig("B", pandar64_beams(), 1800, n_phi=16,
                           pose_end=pose(yaw_quat(0.03), [1.0, 0.0, 1.8]))
    if name == "C":
        return LidarConfig("C", waymo_top_beams(), 2650, n_phi=16,
                           pose_end=pose(yaw_quat(0.02), [1.5, 0.0, 1.8]))
    if name == "tiny":
        return LidarConfig("tiny", uniform_beams(8, -20.0, 10.0), 64, n_phi=4, max_rays_per_tile=16,
                           cull_az_cells=256, pose_end=pose(yaw_quat(0.05), [0.5, 0.2, 1.8]))
    raise ValueError(name)


def camera_config(name: str = "D") -> CameraConfig:
    if name == "D":
        cfg = CameraConfig("D", 1, 1920, 1080, 600.0, 600.0, 960.0, 540.0,
                           (-0.04, 0.004, -0.0006, 0.00004, 0.0))
        cfg.pose_end = pose(yaw_quat(0.009, CAM_FORWARD_Q), [1.8, 0.0, 1.6])
        return cfg
    if name == "D-small":  # same lens scaled down (parity-test size)
        cfg = CameraConfig("D-small", 1, 320, 180, 100.0, 100.0, 160.0, 90.0,
                           (-0.04, 0.004, -0.0006, 0.00004, 0.0))
        cfg.pose_end = pose(yaw_quat(0.009, CAM_FORWARD_Q), [1.8, 0.0, 1.6])
        return cfg
    if name == "pinhole-small":
        cfg = CameraConfig("pinhole-small", 0, 320, 240, 250.0, 250.0, 160.0, 120.0,
                           (-0.1, 0.01, 0.001, -0.0005, 0.0), max_theta=math.radians(50.0))
        cfg.pose_end = pose(yaw_quat(0.01, CAM_FORWARD_Q), [1.8, 0.1, 1.6])
        return cfg
    raise ValueError(name)


# ------------------------------------------------------------------------------------
# scenes
# ------------------------------------------------------------------------------------


def _logu(rng, lo, hi, size):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size))


def _random_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q  # need not be unit (the ABI normalises)


def _yaw_quats(rng, n):
    yaw = rng.uniform(-math.pi, math.pi, n)
    return np.stack([np.cos(yaw / 2), np.zeros(n), np.zeros(n), np.sin(yaw / 2)], 1)


def _axis_normal_quats(rng, n, normal_axis):
    """Rotations taking local z (the thin axis) to world ``normal_axis`` with a random
    in-plane angle."""
    ang = rng.uniform(-math.pi, math.pi, n)
    qin = np.stack([np.cos(ang / 2), np.zeros(n), np.zeros(n), np.sin(ang / 2)], 1)  # about local z
    if normal_axis == "z":
        return qin
    # local z -> world y : rotation of -90 deg about x : (cos45, -sin45, 0, 0)
    base = np.array([math.cos(math.pi / 4), -math.sin(math.pi / 4), 0.0, 0.0])
    w1, x1, y1, z1 = base
    w2, x2, y2, z2 = qin.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], 1)


def _sh_lidar(rng, n):
    sh = rng.normal(0.0, 0.05, size=(n, 16, 3))
    sh[:, 0, 0] = rng.uniform(0.0, 1.0, n) / Y00          # intensity in [0, 1]
    sh[:, 0, 1] = rng.normal(2.0, 1.0, n) / Y00           # hit logit
    sh[:, 0, 2] = rng.normal(-2.0, 1.0, n) / Y00          # drop logit
    return sh


def _sh_camera(rng, n):
    sh = rng.normal(0.0, 0.05, size=(n, 16, 3))
    sh[:, 0, :] = rng.uniform(0.0, 1.0, (n, 3)) / Y00
    return sh


def _pack(means, quats, scales, opac, sh):
    return {
        "means": np.ascontiguousarray(means, np.float32),
        "quats": np.ascontiguousarray(quats, np.float32),
        "scales": np.ascontiguousarray(scales, np.float32),
        "opacity": np.ascontiguousarray(opac, np.float32),
        "sh": np.ascontiguousarray(sh, np.float32).reshape(-1, 16, 3),
    }


def random_shell_scene(seed: int, n: int, center=(0.0, 0.0, 1.8), r_lo=2.0, r_hi=30.0,
                       el_lo=-35.0, el_hi=15.0, s_lo=0.05, s_hi=0.5) -> dict:
    """Config A: uniform in a spherical shell around the sensor."""
    rng = np.random.default_rng(seed)
    r = rng.uniform(r_lo, r_hi, n)
    az = rng.uniform(-math.pi, math.pi, n)
    el = np.radians(rng.uniform(el_lo, el_hi, n))
    means = np.stack([r * np.cos(el) * np.cos(az), r * np.cos(el) * np.sin(az), r * np.sin(el)], 1)
    means += np.asarray(center)
    scales = _logu(rng, s_lo, s_hi, (n, 3))
    quats = _random_quats(rng, n)
    opac = rng.uniform(0.05, 0.99, n)
    sh = rng.normal(0.0, 0.3, size=(n, 16, 3))
    return _pack(means, quats, scales, opac, sh)


def corridor_scene(seed: int, n: int, x_range=(-100.0, 100.0), kind: str = "lidar",
                   ego=(0.0, 0.0, 1.8)) -> dict:
    """Driving corridor: ground, facades, cars, poles, trees,
    floaters.  kind='lidar' -> bimodal opacity + intensity/ray-drop SH; 'camera' ->
    volumetric opacity + colour SH."""
    rng = np.random.default_rng(seed)
    x0, x1 = x_range
    length = x1 - x0
    parts = {"ground": 0.40, "facade": 0.25, "car": 0.10, "pole": 0.05, "tree": 0.15, "float": 0.05}
    counts = {k: int(round(v * n)) for k, v in parts.items()}
    counts["ground"] += n - sum(counts.values())
    M, Q, S = [], [], []

    # ground: z = 0, y in [-30, 30]
    m = counts["ground"]
    M.append(np.stack([rng.uniform(x0, x1, m), rng.uniform(-30, 30, m), np.zeros(m)], 1))
    Q.append(_axis_normal_quats(rng, m, "z"))
    S.append(np.concatenate([_logu(rng, 0.03, 0.12, (m, 2)), _logu(rng, 0.01, 0.02, (m, 1))], 1))

    # facades: y = +-15, z in [0, 20], thin along y
    m = counts["facade"]
    side = np.where(rng.uniform(size=m) < 0.5, -15.0, 15.0)
    M.append(np.stack([rng.uniform(x0, x1, m), side + rng.normal(0, 0.02, m), rng.uniform(0, 20, m)], 1))
    Q.append(_axis_normal_quats(rng, m, "y"))
    S.append(np.concatenate([_logu(rng, 0.03, 0.12, (m, 2)), _logu(rng, 0.01, 0.02, (m, 1))], 1))

    # cars: 4.5 x 1.9 x 1.6 boxes at |y| in [3, 10] (per 200 m: 40 cars)
    m = counts["car"]
    ncar = max(1, int(round(40 * length / 200.0)))
    cx = rng.uniform(x0 + 3, x1 - 3, ncar)
    cy = rng.uniform(3.0, 10.0, ncar) * np.where(rng.uniform(size=ncar) < 0.5, -1, 1)
    which = rng.integers(0, ncar, m)
    face = rng.integers(0, 5, m)  # 0..3 sides, 4 roof
    u, v = rng.uniform(-0.5, 0.5, m), rng.uniform(-0.5, 0.5, m)
    lx, ly, lz = 4.5, 1.9, 1.6
    px = np.where(face == 0, 0.5 * lx, np.where(face == 1, -0.5 * lx, u * lx))
    py = np.where(face == 2, 0.5 * ly, np.where(face == 3, -0.5 * ly, np.where(face < 2, u * ly, v * ly)))
    pz = np.where(face == 4, lz, (v + 0.5) * lz)
    M.append(np.stack([cx[which] + px, cy[which] + py, pz], 1))
    Q.append(_random_quats(rng, m))
    S.append(np.concatenate([_logu(rng, 0.03, 0.10, (m, 2)), _logu(rng, 0.01, 0.02, (m, 1))], 1))

    # poles: r 0.15 m, h 6 m, |y| in [10, 14] (80 per 200 m)
    m = counts["pole"]
    npole = max(1, int(round(80 * length / 200.0)))
    qx = rng.uniform(x0, x1, npole)
    qy = rng.uniform(10.0, 14.0, npole) * np.where(rng.uniform(size=npole) < 0.5, -1, 1)
    which = rng.integers(0, npole, m)
    ang = rng.uniform(-math.pi, math.pi, m)
    M.append(np.stack([qx[which] + 0.15 * np.cos(ang), qy[which] + 0.15 * np.sin(ang), rng.uniform(0, 6, m)], 1))
    Q.append(_random_quats(rng, m))
    S.append(_logu(rng, 0.02, 0.06, (m, 3)))

    # trees: isotropic clusters (30 per 200 m), crowns at 3-7 m, |y| in [16, 25]
    m = counts["tree"]
    ntree = max(1, int(round(30 * length / 200.0)))
    tx = rng.uniform(x0, x1, ntree)
    ty = rng.uniform(16.0, 25.0, ntree) * np.where(rng.uniform(size=ntree) < 0.5, -1, 1)
    tz = rng.uniform(3.0, 7.0, ntree)
    which = rng.integers(0, ntree, m)
    M.append(np.stack([tx[which], ty[which], tz[which]], 1) + rng.normal(0, 1.5, (m, 3)))
    Q.append(_random_quats(rng, m))
    S.append(_logu(rng, 0.05, 0.3, (m, 3)))

    # floaters
    m = counts["float"]
    M.append(np.stack([rng.uniform(x0, x1, m), rng.uniform(-30, 30, m), rng.uniform(0, 20, m)], 1))
    Q.append(_random_quats(rng, m))
    S.append(_logu(rng, 0.05, 0.3, (m, 3)))

    means = np.concatenate(M)
    quats = np.concatenate(Q)
    scales = np.concatenate(S)
    n_tot = means.shape[0]
    is_ground = np.zeros(n_tot, bool)
    is_ground[: counts["ground"]] = True
    # keep the ego lane |y| < 2 free of non-ground particles; nothing within 3 m of the ego
    bad = (~is_ground) & (np.abs(means[:, 1]) < 2.0)
    bad |= np.linalg.norm(means - np.asarray(ego), axis=1) < 3.0
    if bad.any():  # re-draw offending particles as ground particles away from the ego
        k = int(bad.sum())
        gx = rng.uniform(x0, x1, k)
        gy = rng.uniform(3.0, 30.0, k) * np.where(rng.uniform(size=k) < 0.5, -1, 1)
        means[bad] = np.stack([gx, gy, np.zeros(k)], 1)
        quats[bad] = _axis_normal_quats(rng, k, "z")
        scales[bad] = np.concatenate([_logu(rng, 0.03, 0.12, (k, 2)), _logu(rng, 0.01, 0.02, (k, 1))], 1)
    if kind == "lidar":
        hi = rng.uniform(size=n_tot) < 0.85
        opac = np.where(hi, rng.uniform(0.9, 0.99, n_tot), rng.uniform(0.01, 0.2, n_tot))
        sh = _sh_lidar(rng, n_tot)
    else:
        opac = rng.uniform(0.05, 0.99, n_tot)
        sh = _sh_camera(rng, n_tot)
    perm = rng.permutation(n_tot)  # unordered set
    return _pack(means[perm], quats[perm], scales[perm], opac[perm], sh[perm])


def scene_for(config: str, seed: int | None = None, n: int | None = None) -> dict:
    """Scene of a BASELINE.json config: A (1k shell), B (2M corridor), C (4M corridor,
    x in [-200, 200]), D (2M camera corridor), tiny (<=500)."""
    if config == "A":
        return random_shell_scene(1001 if seed is None else seed, n or 1000)
    if config == "B":
        return corridor_scene(1002 if seed is None else seed, n or 2_000_000)
    if config == "C":
        return corridor_scene(1003 if seed is None else seed, n or 4_000_000, x_range=(-200.0, 200.0))
    if config == "D":
        return corridor_scene(1004 if seed is None else seed, n or 2_000_000, kind="camera", ego=(1.5, 0.0, 1.6))
    if config == "E-lidar":  # config E: one 4M G_l + 4M G_c corridor scene, x in [-200, 200]
        return corridor_scene(1005 if seed is None else seed, n or 4_000_000, x_range=(-200.0, 200.0))
    if config == "E-camera":
        return corridor_scene(1006 if seed is None else seed, n or 4_000_000, x_range=(-200.0, 200.0),
                              kind="camera", ego=(1.5, 0.0, 1.6))
    if config == "tiny":
        s = 0 if seed is None else seed
        rng = np.random.default_rng(10_000 + s)
        return random_shell_scene(s, n or int(rng.integers(50, 500)), r_lo=1.0, r_hi=12.0,
                                  el_lo=-30.0, el_hi=20.0, s_lo=0.03, s_hi=0.6)
    raise ValueError(config)


def e_poses(n: int = 64):
    """Config E: n poses along x = -32 .. +31 m (1 m steps, yaw +-0.02
    alternating); scan i is C-type with 1.5 m / 0.02 rad of intra-scan motion, frame i is
    D-type (rolling shutter over 30 ms: +0.3 m, +0.009 rad) from the same pose."""
    scans, frames = [], []
    for i in range(n):
        x = -32.0 + i
        yaw = 0.02 * (1 if i % 2 else -1)
        scans.append((pose(yaw_quat(yaw), [x, 0.0, 1.8]), pose(yaw_quat(yaw + 0.02), [x + 1.5, 0.0, 1.8])))
        frames.append((pose(yaw_quat(yaw, CAM_FORWARD_Q), [x + 1.5, 0.0, 1.6]),
                       pose(yaw_quat(yaw + 0.009, CAM_FORWARD_Q), [x + 1.8, 0.0, 1.6])))
    return scans, frames


def batch_poses(n_scans: int, x_lo: float = -51.0, step: float = 0.2, motion: float = 1.0,
                yaw_rate: float = 0.03, z: float = 1.8):
    """B-batch: scans at poses `step` apart along x, each with `motion` m
    of intra-scan travel and `yaw_rate` rad of yaw."""
    out = []
    for i in range(n_scans):
        x = x_lo + step * i
        yaw0 = 0.01 * ((i % 2) * 2 - 1)
        out.append((pose(yaw_quat(yaw0), [x, 0.0, z]), pose(yaw_quat(yaw0 + yaw_rate), [x + motion, 0.0, z])))
    return out


def with_actors(scene: dict, seed: int, n_actors: int = 8, per_actor: int = 1500, x_range=(5.0, 40.0),
                kind: str = "lidar", yaw_only: bool = False) -> dict:
    """Scene graph input (A29): appends n_actors dynamic objects (car-sized shells
    of per_actor particles each, generated directly in the object's local frame: x forward,
    z up, origin at the box's ground centre) plus their object -> world poses at t (on the
    road at |y| in [3, 9], random yaw, small roll / pitch unless yaw_only).  The static
    scene's particles get actor_id -1.  Returns a new dict with 'actor_id' [n] int32 and
    'actor_pose' [n_actors, 7] float32 (q w,x,y,z, t).  No method arithmetic: the local
    particles and the poses are drawn independently."""
    rng = np.random.default_rng(seed)
    m = n_actors * per_actor
    face = rng.integers(0, 5, m)
    u, v = rng.uniform(-0.5, 0.5, m), rng.uniform(-0.5, 0.5, m)
    lx, ly, lz = 4.5, 1.9, 1.6
    px = np.where(face == 0, 0.5 * lx, np.where(face == 1, -0.5 * lx, u * lx))
    py = np.where(face == 2, 0.5 * ly, np.where(face == 3, -0.5 * ly, np.where(face < 2, u * ly, v * ly)))
    pz = np.where(face == 4, lz, (v + 0.5) * lz)
    means = np.stack([px, py, pz], 1)
    quats = _random_quats(rng, m)
    scales = np.concatenate([_logu(rng, 0.03, 0.10, (m, 2)), _logu(rng, 0.01, 0.02, (m, 1))], 1)
    if kind == "lidar":
        hi = rng.uniform(size=m) < 0.85
        opac = np.where(hi, rng.uniform(0.9, 0.99, m), rng.uniform(0.01, 0.2, m))
        sh = _sh_lidar(rng, m)
    else:
        opac = rng.uniform(0.05, 0.99, m)
        sh = _sh_camera(rng, m)
    ids = np.repeat(np.arange(n_actors, dtype=np.int32), per_actor)
    yaw = rng.uniform(-math.pi, math.pi, n_actors)
    tilt = np.zeros((n_actors, 2)) if yaw_only else rng.normal(0.0, 0.03, (n_actors, 2))
    poses = np.zeros((n_actors, 7), np.float64)
    for a in range(n_actors):  # q = q_z(yaw) q_y(pitch) q_x(roll), composed by hand
        cz, sz = math.cos(yaw[a] / 2), math.sin(yaw[a] / 2)
        cy, sy = math.cos(tilt[a, 1] / 2), math.sin(tilt[a, 1] / 2)
        cx, sx = math.cos(tilt[a, 0] / 2), math.sin(tilt[a, 0] / 2)
        poses[a, :4] = (cz * cy * cx + sz * sy * sx, cz * cy * sx - sz * sy * cx,
                        cz * sy * cx + sz * cy * sx, sz * cy * cx - cz * sy * sx)
    poses[:, 4] = rng.uniform(*x_range, n_actors)
    poses[:, 5] = rng.uniform(3.0, 9.0, n_actors) * np.where(rng.uniform(size=n_actors) < 0.5, -1, 1)
    poses[:, 6] = rng.uniform(-0.05, 0.05, n_actors)
    n0 = scene["means"].shape[0]
    out = {k: np.concatenate([scene[k], v.astype(np.float32).reshape((-1,) + scene[k].shape[1:])])
           for k, v in (("means", means), ("quats", quats), ("scales", scales), ("opacity", opac), ("sh", sh))}
    out["actor_id"] = np.concatenate([np.full(n0, -1, np.int32), ids])
    out["actor_pose"] = poses.astype(np.float32)
    perm = rng.permutation(n0 + m)  # unordered set
    for k in ("means", "quats", "scales", "opacity", "sh", "actor_id"):
        out[k] = np.ascontiguousarray(out[k][perm])
    return out
