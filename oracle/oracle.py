"""ctypes front-end of the CPU oracle (oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this module.  It never imports the product package
(paper_2510_12901_b200) and the product never imports it.  Inputs are plain numpy arrays
(the seeded generators of paper_2510_12901_b200.synth produce them; that module holds no
arithmetic of the method).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C, double, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared",
                               "-fPIC", "-o", LIB_PATH, SRC, "-lm"])
    return LIB_PATH


_lib = None

f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


class OrLidar(C.Structure):
    _fields_ = [("n_beams", C.c_int32), ("elev", f32p), ("n_az", C.c_int32), ("az_start", C.c_double),
                ("dir", C.c_int32), ("r_min", C.c_double), ("beam_div", C.c_double)]


class OrCamera(C.Structure):
    _fields_ = [("model", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double), ("k", C.c_double * 5),
                ("rolling", C.c_int32), ("near_m", C.c_double), ("max_theta", C.c_double),
                ("tile_px", C.c_int32)]


class OrTiling(C.Structure):
    _fields_ = [("n_phi", C.c_int32), ("n_theta", C.c_int32), ("n_tiles", C.c_int32),
                ("max_rays_in_tile", C.c_int32), ("sat_rows", C.c_int32), ("sat_cols", C.c_int32),
                ("n_rays", C.c_int32), ("cull_rows_per_tile", C.c_int32), ("cull_az_cells", C.c_int32),
                ("pi_f", C.c_float), ("two_pi_f", C.c_float), ("az_tile_scale", C.c_float),
                ("az_cell_scale", C.c_float), ("bounds", f32p), ("cull_row_scale", f32p), ("ray_az", f32p),
                ("ray_el", f32p), ("ray_s", f32p), ("ray_tile", i32p), ("tile_ray_offsets", i32p),
                ("tile_rays", i32p), ("sat", i32p), ("ray_cell_row", i32p), ("ray_cell_col", i32p),
                ("n_beams", C.c_int32), ("n_az", C.c_int32)]


class OrProjOut(C.Structure):
    _fields_ = [("valid", i32p), ("ambiguous", i32p), ("mean2d", f64p), ("cov2d", f64p), ("box", f32p),
                ("Mrows", f64p), ("feat", f64p), ("key", f32p), ("minrange", f64p), ("viewdir", f64p)]


class OrGaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", f32p), ("quats", f32p), ("scales", f32p), ("opacity", f32p),
                ("sh", f32p), ("sh_degree", C.c_int32)]


class OrRenderParams(C.Structure):
    _fields_ = [("near_tau", C.c_double), ("alpha_min", C.c_double), ("alpha_max", C.c_double),
                ("T_min", C.c_double), ("wrap", C.c_int32), ("pi_f", C.c_float), ("two_pi_f", C.c_float),
                ("flag_mode", C.c_int32), ("eps_a", C.c_double), ("eps_b", C.c_double),
                ("eps_alpha", C.c_double), ("eps_T_rel", C.c_double), ("eps_tau", C.c_double),
                ("eps_impact", C.c_double), ("eps_amb_a", C.c_double), ("eps_amb_b", C.c_double),
                ("sh", C.c_void_p), ("sh_degree", C.c_int32)]


class OrRenderOut(C.Structure):
    _fields_ = [("feat", f64p), ("opacity", f64p), ("depth_accum", f64p), ("depth", f64p), ("T_final", f64p),
                ("n_contrib", i32p), ("flag", i32p), ("scanned", i64p), ("inbox", i64p)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.or_build_tiling.argtypes = [C.POINTER(OrLidar), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(OrTiling)]
        L.or_free_tiling.argtypes = [C.POINTER(OrTiling)]
        L.or_project_lidar.argtypes = [C.POINTER(OrGaussians), C.POINTER(OrLidar), f64p, f64p, C.c_int, f64p,
                                       C.c_double, C.POINTER(OrProjOut)]
        L.or_project_camera.argtypes = [C.POINTER(OrGaussians), C.POINTER(OrCamera), f64p, f64p, C.c_int, f64p,
                                        C.c_double, C.POINTER(OrProjOut)]
        L.or_cull_lidar.argtypes = [C.c_int64, i32p, f32p, C.POINTER(OrTiling), C.c_int, i32p, i32p]
        L.or_cull_camera.argtypes = [C.c_int64, i32p, f32p, C.POINTER(OrCamera), i32p, i32p]
        L.or_bin.argtypes = [C.c_int64, i32p, i32p, f32p, C.c_int32, C.c_int32, C.c_int64, u64p, u32p, i32p]
        L.or_bin.restype = C.c_int64
        L.or_composite.argtypes = [C.c_int64, f64p, f64p, f64p, f64p, f32p, i32p, u32p, i32p, C.c_int32, i32p,
                                   f32p, f32p, f64p, i32p, C.POINTER(OrRenderParams), C.POINTER(OrRenderOut)]
        L.or_lidar_rays.argtypes = [C.POINTER(OrTiling), f64p, f64p, f64p]
        L.or_camera_rays.argtypes = [C.POINTER(OrCamera), f64p, f64p, f64p, i32p, f32p, f32p, i32p]
        L.or_quat_to_rot.argtypes = [f64p, f64p]
        L.or_covariance.argtypes = [f64p, f64p, f64p]
        L.or_sigma_points.argtypes = [f64p, f64p, f64p, f64p, f64p, f64p, f64p]
        L.or_pose_at.argtypes = [f64p, f64p, C.c_double, f64p, f64p]
        L.or_lidar_point.argtypes = [f64p, C.POINTER(OrLidar), f64p, f64p, C.c_int, f64p]
        L.or_camera_point.argtypes = [f64p, C.POINTER(OrCamera), f64p, f64p, C.c_int, f64p]
        L.or_camera_unproject.argtypes = [C.POINTER(OrCamera), C.c_double, C.c_double, f64p]
        L.or_sh_eval.argtypes = [f64p, C.c_int, f64p, f64p]
        L.or_response.argtypes = [f64p, f64p, f64p, f64p, f64p]
        L.or_ut_affine.argtypes = [f64p, f64p, f64p, f64p, f64p, f64p, f64p, f64p]
        L.or_compose_camera.argtypes = [C.POINTER(OrCamera), f64p, f64p, f64p, f32p, C.c_int32, C.c_int32, f32p,
                                        C.c_int32, C.c_int32, C.c_int32, f64p]
        L.or_divergence_cov.argtypes = [f64p, f64p, f64p, C.c_double, f64p]
        L.or_cholesky3.argtypes = [f64p, f64p]
        L.or_lower_inverse3.argtypes = [f64p, f64p]
        L.or_sigma_points_sqrt.argtypes = [f64p, f64p, f64p, f64p, f64p, f64p]
        L.or_sat_query.argtypes = [i32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.or_decode_lidar.argtypes = [f64p, f64p]
        L.or_elev_tile.argtypes = [C.POINTER(OrTiling), C.c_float]
        L.or_az_col.argtypes = [C.POINTER(OrTiling), C.c_float]
        L.or_set_threads.argtypes = [C.c_int]
        L.or_backward_composite.argtypes = [f64p, f64p, f64p, f64p, f32p, u32p, i32p, C.c_int32, i32p, f32p, f32p,
                                            f64p, i32p, C.POINTER(OrRenderParams), f64p, f64p, f64p, f64p, f64p,
                                            f64p, f64p, f64p]
        L.or_backward_params_sg.argtypes = [C.c_int64, f32p, f32p, f32p, f64p, C.c_int32, i32p, C.c_int32, f64p,
                                            C.c_double, f64p, f64p, f64p, f64p, f64p, f64p, f64p, f64p]
        L.or_actors_to_world.argtypes = [C.c_int64, f32p, f32p, i32p, C.c_int32, f64p, f32p, f32p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _d(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def set_threads(n: int):
    lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(lib().or_get_threads())


# ------------------------------------------------------------------------------------
# sensor / pose marshalling (float32 ABI values promoted to double)
# ------------------------------------------------------------------------------------

def pose7(p) -> np.ndarray:
    q = np.asarray(p["q"], np.float32).astype(np.float64)
    t = np.asarray(p["t"], np.float32).astype(np.float64)
    return np.concatenate([q, t])


def make_lidar(cfg):
    beams = np.ascontiguousarray(cfg.beams, np.float32)
    L = OrLidar(int(beams.shape[0]), _p(beams, f32p), int(cfg.n_azimuth), float(np.float32(cfg.azimuth_start)),
                int(cfg.spin_direction), float(np.float32(cfg.min_range)),
                float(np.float32(getattr(cfg, "beam_divergence", 0.0))))
    L._keep = beams
    return L


def make_camera(cfg):
    k = (C.c_double * 5)(*[float(np.float32(x)) for x in cfg.k])
    f = lambda x: float(np.float32(x))  # noqa: E731
    return OrCamera(int(cfg.model), int(cfg.width), int(cfg.height), f(cfg.fx), f(cfg.fy), f(cfg.cx), f(cfg.cy), k,
                    int(cfg.rolling_shutter), f(cfg.near), f(cfg.max_theta), int(cfg.tile_px))


# ------------------------------------------------------------------------------------
# O7 tiling
# ------------------------------------------------------------------------------------

class Tiling:
    """Owns an or_tiling; exposes numpy copies of every array."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.L = make_lidar(cfg)
        self.t = OrTiling()
        rc = lib().or_build_tiling(C.byref(self.L), cfg.n_phi, cfg.max_rays_per_tile, cfg.hist_bins,
                                   cfg.cull_az_cells, cfg.cull_rows_per_tile, C.byref(self.t))
        if rc != 0:
            raise ValueError(f"or_build_tiling failed ({rc})")
        t = self.t
        R = t.n_rays
        cp = lambda ptr, n: np.ctypeslib.as_array(ptr, shape=(n,)).copy()  # noqa: E731
        self.n_phi, self.n_theta, self.n_tiles = t.n_phi, t.n_theta, t.n_tiles
        self.max_rays_in_tile, self.sat_rows, self.sat_cols = t.max_rays_in_tile, t.sat_rows, t.sat_cols
        self.pi_f, self.two_pi_f = np.float32(t.pi_f), np.float32(t.two_pi_f)
        self.az_tile_scale, self.az_cell_scale = np.float32(t.az_tile_scale), np.float32(t.az_cell_scale)
        self.bounds = cp(t.bounds, t.n_phi + 1)
        self.cull_row_scale = cp(t.cull_row_scale, t.n_phi)
        self.ray_az, self.ray_el, self.ray_s = cp(t.ray_az, R), cp(t.ray_el, R), cp(t.ray_s, R)
        self.ray_tile = cp(t.ray_tile, R)
        self.tile_ray_offsets = cp(t.tile_ray_offsets, t.n_tiles + 1)
        self.tile_rays = cp(t.tile_rays, R)
        self.sat = cp(t.sat, t.sat_rows * t.sat_cols).reshape(t.sat_rows, t.sat_cols)
        self.ray_cell_row, self.ray_cell_col = cp(t.ray_cell_row, R), cp(t.ray_cell_col, R)
        self.n_rays = R

    def elev_tile(self, w):
        return lib().or_elev_tile(C.byref(self.t), C.c_float(w))

    def az_col(self, phi):
        return lib().or_az_col(C.byref(self.t), C.c_float(phi))

    def __del__(self):
        try:
            lib().or_free_tiling(C.byref(self.t))
        except Exception:
            pass


# ------------------------------------------------------------------------------------
# projection
# ------------------------------------------------------------------------------------

def _gauss(scene):
    if scene.get("actor_id") is not None:  # scene graph first (O0)
        scene = actors_to_world(scene)
    n = int(scene["means"].shape[0])
    arrs = {k: np.ascontiguousarray(scene[k], np.float32) for k in ("means", "quats", "scales", "opacity", "sh")}
    ncoef = arrs["sh"].size // max(n, 1) // 3 if n else 16
    deg = {1: 0, 4: 1, 9: 2, 16: 3}[ncoef]  # SH degree from the coefficient count
    G = OrGaussians(n, _p(arrs["means"], f32p), _p(arrs["quats"], f32p), _p(arrs["scales"], f32p),
                    _p(arrs["opacity"], f32p), _p(arrs["sh"], f32p), deg)
    G._keep = arrs
    return G, n


def _proj_out(n):
    o = {"valid": np.zeros(n, np.int32), "ambiguous": np.zeros(n, np.int32), "mean2d": np.zeros((n, 2)),
         "cov2d": np.zeros((n, 3)), "box": np.zeros((n, 4), np.float32), "Mrows": np.zeros((n, 9)),
         "feat": np.zeros((n, 3)), "key": np.zeros(n, np.float32), "minrange": np.zeros(n),
         "viewdir": np.zeros((n, 3))}
    s = OrProjOut(_p(o["valid"], i32p), _p(o["ambiguous"], i32p), _p(o["mean2d"], f64p), _p(o["cov2d"], f64p),
                  _p(o["box"], f32p), _p(o["Mrows"], f64p), _p(o["feat"], f64p), _p(o["key"], f32p),
                  _p(o["minrange"], f64p), _p(o["viewdir"], f64p))
    return o, s


def _ut(ut):
    return _d(ut if ut is not None else (1.0, 2.0, 0.0))


def project_lidar(scene, cfg, pose0=None, pose1=None, K=None, ut=None, extent_sigma=3.0):
    G, n = _gauss(scene)
    L = make_lidar(cfg)
    p0 = pose7(pose0 or cfg.pose_start)
    p1 = pose7(pose1 or cfg.pose_end)
    o, s = _proj_out(n)
    u = _ut(ut)
    rc = lib().or_project_lidar(C.byref(G), C.byref(L), _p(p0, f64p), _p(p1, f64p),
                                cfg.rs_iterations if K is None else K, _p(u, f64p), extent_sigma, C.byref(s))
    assert rc == 0
    return o


def project_camera(scene, cam, pose0=None, pose1=None, K=None, ut=None, extent_sigma=3.0):
    G, n = _gauss(scene)
    Cm = make_camera(cam)
    p0 = pose7(pose0 or cam.pose_start)
    p1 = pose7(pose1 or cam.pose_end)
    o, s = _proj_out(n)
    u = _ut(ut)
    rc = lib().or_project_camera(C.byref(G), C.byref(Cm), _p(p0, f64p), _p(p1, f64p),
                                 cam.rs_iterations if K is None else K, _p(u, f64p), extent_sigma, C.byref(s))
    assert rc == 0
    return o


# ------------------------------------------------------------------------------------
# culling, binning
# ------------------------------------------------------------------------------------

def cull_lidar(valid, box, tiling: Tiling, enable_cull=True):
    """Counts and tile rects (O8).  enable_cull: 0/False off, 1/True the paper's dense-grid
    SAT test (Proc. RayOccupancyCount / ProjectParticles), 2 exact ray containment (A32)."""
    n = int(valid.shape[0])
    valid = np.ascontiguousarray(valid, np.int32)
    box = np.ascontiguousarray(box, np.float32)
    count = np.zeros(n, np.int32)
    rect = np.zeros((n, 4), np.int32)
    rc = lib().or_cull_lidar(n, _p(valid, i32p), _p(box, f32p), C.byref(tiling.t), int(enable_cull),
                             _p(count, i32p), _p(rect, i32p))
    if rc != 0:
        raise RuntimeError("or_cull_lidar: column set is not a single circular run")
    return count, rect


def camera_tiles(cam):
    tp = cam.tile_px
    Wt, Ht = (cam.width + tp - 1) // tp, (cam.height + tp - 1) // tp
    return Wt, Ht


def cull_camera(valid, box, cam):
    n = int(valid.shape[0])
    valid = np.ascontiguousarray(valid, np.int32)
    box = np.ascontiguousarray(box, np.float32)
    count = np.zeros(n, np.int32)
    rect = np.zeros((n, 4), np.int32)
    Cm = make_camera(cam)
    lib().or_cull_camera(n, _p(valid, i32p), _p(box, f32p), C.byref(Cm), _p(count, i32p), _p(rect, i32p))
    return count, rect


def bin_pairs(count, rect, key, n_tiles, n_cols_total):
    n = int(count.shape[0])
    count = np.ascontiguousarray(count, np.int32)
    rect = np.ascontiguousarray(rect, np.int32)
    key = np.ascontiguousarray(key, np.float32)
    P = int(count.astype(np.int64).sum())
    keys = np.zeros(max(P, 1), np.uint64)
    ids = np.zeros(max(P, 1), np.uint32)
    ranges = np.zeros((n_tiles, 2), np.int32)
    P2 = lib().or_bin(n, _p(count, i32p), _p(rect, i32p), _p(key, f32p), n_tiles, n_cols_total, P,
                      _p(keys, u64p), _p(ids, u32p), _p(ranges, i32p))
    assert P2 == P
    return keys[:P], ids[:P], ranges


def sort_all(valid, key):
    """Brute-force list (O13): every valid Gaussian once, ordered by (key, id)."""
    n = int(valid.shape[0])
    count = np.ascontiguousarray((np.asarray(valid) != 0).astype(np.int32))
    rect = np.zeros((n, 4), np.int32)
    rect[:, 3] = 1
    _, ids, ranges = bin_pairs(count, rect, key, 1, 1)
    return ids, ranges


# ------------------------------------------------------------------------------------
# rays + compositing
# ------------------------------------------------------------------------------------

def lidar_rays(tiling: Tiling, pose0, pose1):
    od = np.zeros((tiling.n_rays, 6))
    lib().or_lidar_rays(C.byref(tiling.t), _p(pose7(pose0), f64p), _p(pose7(pose1), f64p), _p(od, f64p))
    return od


def camera_rays(cam, pose0=None, pose1=None):
    n = cam.width * cam.height
    od = np.zeros((n, 6))
    valid = np.zeros(n, np.int32)
    pu = np.zeros(n, np.float32)
    pv = np.zeros(n, np.float32)
    tile = np.zeros(n, np.int32)
    Cm = make_camera(cam)
    lib().or_camera_rays(C.byref(Cm), _p(pose7(pose0 or cam.pose_start), f64p), _p(pose7(pose1 or cam.pose_end), f64p),
                         _p(od, f64p), _p(valid, i32p), _p(pu, f32p), _p(pv, f32p), _p(tile, i32p))
    return {"od": od, "valid": valid, "u": pu, "v": pv, "tile": tile}


def composite(records, ids, ranges, ray_tile, ray_a, ray_b, ray_od, *, wrap, near, ray_valid=None,
              alpha_min=1.0 / 255.0, alpha_max=0.99, T_min=1e-4, gamb=None, flag_eps=None, pi_f=None,
              two_pi_f=None):
    """records: dict with mu[n,3], Mrows[n,9], sigma[n], feat[n,3] (double) and box[n,4] (float32)."""
    mu = _d(records["mu"])
    Mr = _d(records["Mrows"])
    sg = _d(records["sigma"])
    ft = _d(records["feat"])
    box = np.ascontiguousarray(records["box"], np.float32)
    ids = np.ascontiguousarray(ids, np.uint32)
    ranges = np.ascontiguousarray(ranges, np.int32)
    ray_tile = np.ascontiguousarray(ray_tile, np.int32)
    ra = np.ascontiguousarray(ray_a, np.float32)
    rb = np.ascontiguousarray(ray_b, np.float32)
    od = _d(ray_od)
    rv = None if ray_valid is None else np.ascontiguousarray(ray_valid, np.int32)
    ga = None if gamb is None else np.ascontiguousarray(gamb, np.int32)
    R = int(ray_tile.shape[0])
    pf = np.float32(np.pi) if pi_f is None else np.float32(pi_f)
    tpf = np.float32(2 * np.pi) if two_pi_f is None else np.float32(two_pi_f)
    fe = flag_eps or {}
    prm = OrRenderParams(float(np.float32(near)), float(np.float32(alpha_min)), float(np.float32(alpha_max)),
                         float(np.float32(T_min)), int(wrap), pf, tpf, int(flag_eps is not None),
                         fe.get("a", 0.0), fe.get("b", 0.0), fe.get("alpha", 0.0), fe.get("T_rel", 0.0),
                         fe.get("tau", 0.0), fe.get("impact", 0.0), fe.get("amb_a", AMBIGUOUS_MARGIN[0]),
                         fe.get("amb_b", AMBIGUOUS_MARGIN[1]))
    sh = records.get("sh")  # per-ray SH (literal Eq. 1, A30)
    if sh is not None:
        sh = np.ascontiguousarray(sh, np.float32).reshape(mu.shape[0], -1)
        prm.sh = sh.ctypes.data
        prm.sh_degree = {3: 0, 12: 1, 27: 2, 48: 3}[sh.shape[1]]
    out = {"feat": np.zeros((R, 3)), "opacity": np.zeros(R), "depth_accum": np.zeros(R), "depth": np.zeros(R),
           "T_final": np.zeros(R), "n_contrib": np.zeros(R, np.int32), "flag": np.zeros(R, np.int32),
           "scanned": np.zeros(R, np.int64), "inbox": np.zeros(R, np.int64)}
    so = OrRenderOut(_p(out["feat"], f64p), _p(out["opacity"], f64p), _p(out["depth_accum"], f64p),
                     _p(out["depth"], f64p), _p(out["T_final"], f64p), _p(out["n_contrib"], i32p),
                     _p(out["flag"], i32p), _p(out["scanned"], i64p), _p(out["inbox"], i64p))
    lib().or_composite(int(mu.shape[0]), _p(mu, f64p), _p(Mr, f64p), _p(sg, f64p), _p(ft, f64p), _p(box, f32p),
                       _p(ga, i32p), _p(ids, u32p), _p(ranges, i32p), R, _p(ray_tile, i32p), _p(ra, f32p),
                       _p(rb, f32p), _p(od, f64p), _p(rv, i32p), C.byref(prm), C.byref(so))
    return out


def decode_lidar(zeta):
    """(gamma, beta_drop) per ray."""
    zeta = _d(zeta)
    out = np.zeros((zeta.shape[0], 2))
    for i in range(zeta.shape[0]):
        lib().or_decode_lidar(_p(zeta[i], f64p), _p(out[i], f64p))
    return out[:, 0], out[:, 1]


def records_from_projection(proj, scene):
    if scene.get("actor_id") is not None:  # world particles (O0)
        scene = actors_to_world(scene)
    return {"mu": scene["means"].astype(np.float64), "Mrows": proj["Mrows"],
            "sigma": scene["opacity"].astype(np.float64), "feat": proj["feat"], "box": proj["box"]}


# ------------------------------------------------------------------------------------
# whole-path oracle renders (tier 2)
# ------------------------------------------------------------------------------------

AMBIGUOUS_MARGIN = (0.1, 0.02)  # rad: listing margin of validity-ambiguous particles (flag mode)


def expand_box(box, ea, eb):
    """Grow float32 boxes outward by (ea, eb) (flag-mode list construction)."""
    b = box.astype(np.float64)
    out = np.empty_like(box)
    out[:, 0] = np.nextafter((b[:, 0] - ea).astype(np.float32), np.float32(-np.inf))
    out[:, 1] = np.nextafter((b[:, 1] + ea).astype(np.float32), np.float32(np.inf))
    out[:, 2] = np.nextafter((b[:, 2] - eb).astype(np.float32), np.float32(-np.inf))
    out[:, 3] = np.nextafter((b[:, 3] + eb).astype(np.float32), np.float32(np.inf))
    return out


def render_lidar(scene, cfg, tiling: Tiling | None = None, pose0=None, pose1=None, mode="tiled", enable_cull=True,
                 flag_eps=None, alpha_min=1.0 / 255.0, alpha_max=0.99, T_min=1e-4, ut=None, K=None,
                 ray_od=None, proj=None, per_ray_sh=False):
    """Full oracle LiDAR scan (O1-O13).  mode='tiled' (O7-O12) or 'brute' (O13).  With
    flag_eps, lists come from boxes grown by the margins and rays near a threshold are
    flagged (A23).  per_ray_sh: features SH_i(d) at each ray's direction (Eq. 1, A30)."""
    tiling = tiling or Tiling(cfg)
    pose0 = pose0 or cfg.pose_start
    pose1 = pose1 or cfg.pose_end
    if proj is None:
        proj = project_lidar(scene, cfg, pose0, pose1, K=K, ut=ut)
    rec = records_from_projection(proj, scene)
    if per_ray_sh:
        rec["sh"] = scene["sh"]
    valid = proj["valid"]
    gamb = None
    if flag_eps is not None:
        gamb = np.where(proj["ambiguous"] != 0, np.where(valid != 0, 1, 2), 0).astype(np.int32)
        listed = ((valid != 0) | (proj["ambiguous"] != 0)) & np.isfinite(proj["box"]).all(1)
        lbox = expand_box(proj["box"], flag_eps["a"], flag_eps["b"])
        amb = proj["ambiguous"] != 0  # e.g. a sigma point at the sweep seam: the float32 box may differ a lot
        lbox[amb] = expand_box(proj["box"][amb], flag_eps.get("amb_a", AMBIGUOUS_MARGIN[0]),
                               flag_eps.get("amb_b", AMBIGUOUS_MARGIN[1]))
    else:
        listed = valid != 0
        lbox = proj["box"]
    if mode == "tiled":
        count, rect = cull_lidar(listed.astype(np.int32), lbox, tiling, int(enable_cull) if flag_eps is None else 0)
        _, ids, ranges = bin_pairs(count, rect, proj["key"], tiling.n_tiles, tiling.n_theta)
        ray_tile = tiling.ray_tile
    else:
        ids, ranges = sort_all(listed, proj["key"])
        ray_tile = np.zeros(tiling.n_rays, np.int32)
    od = lidar_rays(tiling, pose0, pose1) if ray_od is None else ray_od
    out = composite(rec, ids, ranges, ray_tile, tiling.ray_az, tiling.ray_el, od, wrap=1,
                    near=cfg.min_range, alpha_min=alpha_min, alpha_max=alpha_max, T_min=T_min, gamb=gamb,
                    flag_eps=flag_eps, pi_f=tiling.pi_f, two_pi_f=tiling.two_pi_f)
    gam, bd = decode_lidar(out["feat"])
    out["intensity"] = gam
    out["raydrop"] = bd
    out["proj"] = proj
    out["ray_od"] = od
    return out


def render_camera(scene, cam, pose0=None, pose1=None, mode="tiled", flag_eps=None, alpha_min=1.0 / 255.0,
                  alpha_max=0.99, T_min=1e-4, ut=None, K=None, rays=None, proj=None, per_ray_sh=False):
    pose0 = pose0 or cam.pose_start
    pose1 = pose1 or cam.pose_end
    if proj is None:
        proj = project_camera(scene, cam, pose0, pose1, K=K, ut=ut)
    rec = records_from_projection(proj, scene)
    if per_ray_sh:
        rec["sh"] = scene["sh"]
    valid = proj["valid"]
    gamb = None
    if flag_eps is not None:
        gamb = np.where(proj["ambiguous"] != 0, np.where(valid != 0, 1, 2), 0).astype(np.int32)
        listed = ((valid != 0) | (proj["ambiguous"] != 0)) & np.isfinite(proj["box"]).all(1)
        lbox = expand_box(proj["box"], flag_eps["a"], flag_eps["b"])
        amb = proj["ambiguous"] != 0
        lbox[amb] = expand_box(proj["box"][amb], flag_eps.get("amb_a", 20.0), flag_eps.get("amb_b", 20.0))
    else:
        listed = valid != 0
        lbox = proj["box"]
    Wt, Ht = camera_tiles(cam)
    rays = rays or camera_rays(cam, pose0, pose1)
    if mode == "tiled":
        count, rect = cull_camera(listed.astype(np.int32), lbox, cam)
        _, ids, ranges = bin_pairs(count, rect, proj["key"], Wt * Ht, Wt)
        ray_tile = rays["tile"]
    else:
        ids, ranges = sort_all(listed, proj["key"])
        ray_tile = np.zeros(cam.width * cam.height, np.int32)
    out = composite(rec, ids, ranges, ray_tile, rays["u"], rays["v"], rays["od"], wrap=0, near=cam.near,
                    ray_valid=rays["valid"], alpha_min=alpha_min, alpha_max=alpha_max, T_min=T_min, gamb=gamb,
                    flag_eps=flag_eps)
    out["proj"] = proj
    out["rays"] = rays
    return out


# ------------------------------------------------------------------------------------
# primitives (pins)
# ------------------------------------------------------------------------------------

def quat_to_rot(q):
    R = np.zeros(9)
    lib().or_quat_to_rot(_p(_d(q), f64p), _p(R, f64p))
    return R.reshape(3, 3)


def covariance(q, s):
    S = np.zeros(9)
    lib().or_covariance(_p(_d(q), f64p), _p(_d(s), f64p), _p(S, f64p))
    return S.reshape(3, 3)


def sigma_points(mu, q, s, ut=None):
    pts, wm, wc = np.zeros(21), np.zeros(7), np.zeros(7)
    rc = lib().or_sigma_points(_p(_d(mu), f64p), _p(_d(q), f64p), _p(_d(s), f64p), _p(_ut(ut), f64p),
                               _p(pts, f64p), _p(wm, f64p), _p(wc, f64p))
    assert rc == 0
    return pts.reshape(7, 3), wm, wc


def compose_camera(cam, ray_od, rgb_fg, omega, env=None, grid=None):
    """Eq. 2: c = A(omega c_f + (1 - omega) c_b(d)); env [He, We, 3], grid [gd, gh, gw, 12]."""
    n = cam.width * cam.height
    out = np.zeros((n, 3))
    Cm = make_camera(cam)
    e = None if env is None else np.ascontiguousarray(env, np.float32)
    g = None if grid is None else np.ascontiguousarray(grid, np.float32)
    lib().or_compose_camera(C.byref(Cm), _p(_d(ray_od).reshape(-1), f64p), _p(_d(rgb_fg).reshape(-1), f64p),
                            _p(_d(omega), f64p), None if e is None else _p(e, f32p),
                            0 if e is None else e.shape[0], 0 if e is None else e.shape[1],
                            None if g is None else _p(g, f32p), 0 if g is None else g.shape[1],
                            0 if g is None else g.shape[2], 0 if g is None else g.shape[0], _p(out, f64p))
    return out


# ------------------------------------------------------------------------------------
# backward (O15, O16; reading A31)
# ------------------------------------------------------------------------------------

def fold_upstream(fwd, grads, lidar):
    """Upstream gradients of the decoded outputs -> (G_feat [R,3], G_omega [R], G_D [R]):
    depth = D / omega (omega > 0, else 0), LiDAR intensity = zeta_0, ray drop
    beta = 1 / (1 + exp(zeta_1 - zeta_2))."""
    R = fwd["opacity"].shape[0]
    g = lambda k, shape: (np.zeros(shape) if grads.get(k) is None  # noqa: E731
                          else np.asarray(grads[k], np.float64).reshape(shape).copy())
    Gz = g("rgb" if not lidar else "zeta", (R, 3))
    Go = g("opacity", R)
    GD = g("depth_accum", R)
    gd = g("depth", R)
    om, D = fwd["opacity"], fwd["depth_accum"]
    pos = om > 0
    GD[pos] += gd[pos] / om[pos]
    Go[pos] -= gd[pos] * D[pos] / om[pos] ** 2
    if lidar:
        Gz[:, 0] += g("intensity", R)
        beta = 1.0 / (1.0 + np.exp(fwd["feat"][:, 1] - fwd["feat"][:, 2]))
        gr = g("raydrop", R) * beta * (1.0 - beta)
        Gz[:, 1] -= gr
        Gz[:, 2] += gr
    return Gz, Go, GD


def backward_composite(records, ids, ranges, ray_tile, ray_a, ray_b, ray_od, Gz, Go, GD, *, wrap, near,
                       ray_valid=None, alpha_min=1.0 / 255.0, alpha_max=0.99, T_min=1e-4, pi_f=None, two_pi_f=None):
    """O15: dL/d(mu, M, sigma, f) per particle (double)."""
    n = records["mu"].shape[0]
    pf = np.float32(np.pi) if pi_f is None else np.float32(pi_f)
    tpf = np.float32(2 * np.pi) if two_pi_f is None else np.float32(two_pi_f)
    prm = OrRenderParams(float(np.float32(near)), float(np.float32(alpha_min)), float(np.float32(alpha_max)),
                         float(np.float32(T_min)), int(wrap), pf, tpf, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    out = {"mu": np.zeros((n, 3)), "M": np.zeros((n, 9)), "sigma": np.zeros(n), "feat": np.zeros((n, 3))}
    sh = records.get("sh")  # per-ray SH (A30): dL/dSH accumulated per (ray, particle)
    if sh is not None:
        sh = np.ascontiguousarray(sh, np.float32).reshape(n, -1)
        prm.sh = sh.ctypes.data
        prm.sh_degree = {3: 0, 12: 1, 27: 2, 48: 3}[sh.shape[1]]
        out["sh_perray"] = np.zeros((n, sh.shape[1] // 3, 3))
    mu, Mr, sg, ft = _d(records["mu"]), _d(records["Mrows"]), _d(records["sigma"]), _d(records["feat"])
    box = np.ascontiguousarray(records["box"], np.float32)
    ids = np.ascontiguousarray(ids, np.uint32)
    ranges = np.ascontiguousarray(ranges, np.int32)
    rt = np.ascontiguousarray(ray_tile, np.int32)
    ra, rb = np.ascontiguousarray(ray_a, np.float32), np.ascontiguousarray(ray_b, np.float32)
    rv = None if ray_valid is None else np.ascontiguousarray(ray_valid, np.int32)
    od, Gz, Go, GD = _d(ray_od), _d(Gz), _d(Go), _d(GD)
    rc = lib().or_backward_composite(_p(mu, f64p), _p(Mr, f64p), _p(sg, f64p), _p(ft, f64p), _p(box, f32p),
                                     _p(ids, u32p), _p(ranges, i32p), int(rt.shape[0]), _p(rt, i32p), _p(ra, f32p),
                                     _p(rb, f32p), _p(od, f64p), _p(rv, i32p), C.byref(prm), _p(Gz, f64p),
                                     _p(Go, f64p), _p(GD, f64p), _p(out["mu"], f64p), _p(out["M"], f64p),
                                     _p(out["sigma"], f64p), _p(out["feat"], f64p), _p(out.get("sh_perray"), f64p))
    assert rc == 0
    return out


def backward_params(scene, proj, d, beam_div=0.0):
    """O16: gradients of the particle parameters (means, quats, scales, opacity, sh); with a
    scene graph the object-frame ones plus the object poses ('actor_pose' [n_actors, 7]:
    dq_a, dt_a); with beam divergence (theta > 0) through Sigma_hat's Cholesky inverse.
    proj['viewdir'] is the view vector mu - o (unnormalised)."""
    n = int(scene["means"].shape[0])
    m = np.ascontiguousarray(scene["means"], np.float32)
    q = np.ascontiguousarray(scene["quats"], np.float32)
    s = np.ascontiguousarray(scene["scales"], np.float32)
    act = scene.get("actor_id")
    ids = None if act is None else np.ascontiguousarray(act, np.int32)
    ap = None if act is None else _d(np.asarray(scene["actor_pose"], np.float32).astype(np.float64))
    na = 0 if ap is None else int(ap.shape[0])
    ncoef = scene["sh"].size // max(n, 1) // 3
    deg = {1: 0, 4: 1, 9: 2, 16: 3}[ncoef]
    out = {"means": np.zeros((n, 3)), "quats": np.zeros((n, 4)), "scales": np.zeros((n, 3)),
           "sh": np.zeros((n, ncoef, 3))}
    ga = np.zeros((max(na, 1), 7))
    lib().or_backward_params_sg(n, _p(m, f32p), _p(q, f32p), _p(s, f32p), _p(_d(proj["viewdir"]), f64p), deg,
                                _p(ids, i32p), na, _p(ap, f64p), float(beam_div), _p(_d(d["mu"]), f64p),
                                _p(_d(d["M"]), f64p), _p(_d(d["feat"]), f64p), _p(out["means"], f64p),
                                _p(out["quats"], f64p), _p(out["scales"], f64p), _p(out["sh"], f64p), _p(ga, f64p))
    if act is not None:
        out["actor_pose"] = ga[:na]
    out["opacity"] = d["sigma"].copy()
    if d.get("sh_perray") is not None:  # per-ray SH: the SH gradient came from O15 directly
        out["sh"] = d["sh_perray"].copy()
    return out


def backward_lidar(scene, cfg, grads, tiling: Tiling | None = None, pose0=None, pose1=None, K=None, ut=None,
                   alpha_min=1.0 / 255.0, alpha_max=0.99, T_min=1e-4, per_ray_sh=False):
    """Whole-path LiDAR backward (O1-O12 forward, O15, O16).  grads: upstream gradients by
    output name (zeta, opacity, depth_accum, depth, intensity, raydrop; missing = 0)."""
    tiling = tiling or Tiling(cfg)
    pose0 = pose0 or cfg.pose_start
    pose1 = pose1 or cfg.pose_end
    fwd = render_lidar(scene, cfg, tiling=tiling, pose0=pose0, pose1=pose1, K=K, ut=ut, alpha_min=alpha_min,
                       alpha_max=alpha_max, T_min=T_min, per_ray_sh=per_ray_sh)
    proj = fwd["proj"]
    rec = records_from_projection(proj, scene)
    if per_ray_sh:
        rec["sh"] = scene["sh"]
    count, rect = cull_lidar(proj["valid"], proj["box"], tiling, True)
    _, ids, ranges = bin_pairs(count, rect, proj["key"], tiling.n_tiles, tiling.n_theta)
    Gz, Go, GD = fold_upstream(fwd, grads, lidar=True)
    d = backward_composite(rec, ids, ranges, tiling.ray_tile, tiling.ray_az, tiling.ray_el, fwd["ray_od"], Gz, Go,
                           GD, wrap=1, near=cfg.min_range, alpha_min=alpha_min, alpha_max=alpha_max, T_min=T_min,
                           pi_f=tiling.pi_f, two_pi_f=tiling.two_pi_f)
    out = backward_params(scene, proj, d, beam_div=getattr(cfg, "beam_divergence", 0.0))
    out["fwd"] = fwd
    out["d"] = d
    return out


def backward_camera(scene, cam, grads, pose0=None, pose1=None, K=None, ut=None, alpha_min=1.0 / 255.0,
                    alpha_max=0.99, T_min=1e-4):
    """Whole-path camera backward; grads keys rgb, opacity, depth_accum, depth."""
    pose0 = pose0 or cam.pose_start
    pose1 = pose1 or cam.pose_end
    fwd = render_camera(scene, cam, pose0=pose0, pose1=pose1, K=K, ut=ut, alpha_min=alpha_min, alpha_max=alpha_max,
                        T_min=T_min)
    proj, rays = fwd["proj"], fwd["rays"]
    rec = records_from_projection(proj, scene)
    Wt, Ht = camera_tiles(cam)
    count, rect = cull_camera(proj["valid"], proj["box"], cam)
    _, ids, ranges = bin_pairs(count, rect, proj["key"], Wt * Ht, Wt)
    Gz, Go, GD = fold_upstream(fwd, grads, lidar=False)
    d = backward_composite(rec, ids, ranges, rays["tile"], rays["u"], rays["v"], rays["od"], Gz, Go, GD, wrap=0,
                           near=cam.near, ray_valid=rays["valid"], alpha_min=alpha_min, alpha_max=alpha_max,
                           T_min=T_min)
    out = backward_params(scene, proj, d)
    out["fwd"] = fwd
    out["d"] = d
    return out


def actors_to_world(scene, actor_id=None, actor_pose=None):
    """O0 (A29): the scene with object particles mapped to world coordinates at t.
    actor_id [n] int32 (-1 static), actor_pose [n_actors, 7] (q w,x,y,z, t); defaults to the
    scene's own 'actor_id' / 'actor_pose' keys.  Returns a new scene dict without them."""
    actor_id = scene.get("actor_id") if actor_id is None else actor_id
    actor_pose = scene.get("actor_pose") if actor_pose is None else actor_pose
    out = {k: v for k, v in scene.items() if k not in ("actor_id", "actor_pose")}
    if actor_id is None:
        return out
    n = int(scene["means"].shape[0])
    m = np.ascontiguousarray(scene["means"], np.float32)
    q = np.ascontiguousarray(scene["quats"], np.float32)
    ids = np.ascontiguousarray(actor_id, np.int32)
    ap = _d(np.asarray(actor_pose, np.float32).astype(np.float64))  # the float32 poses, exactly
    mw, qw = np.zeros((n, 3), np.float32), np.zeros((n, 4), np.float32)
    lib().or_actors_to_world(n, _p(m, f32p), _p(q, f32p), _p(ids, i32p), int(ap.shape[0]), _p(ap, f64p),
                             _p(mw, f32p), _p(qw, f32p))
    out["means"], out["quats"] = mw, qw
    return out


def divergence_cov(Sigma, mu, o, theta):
    """App. C: Sigma_hat = Sigma + (theta r)^2 (I - d d^T)."""
    Sh = np.zeros(9)
    lib().or_divergence_cov(_p(_d(Sigma), f64p), _p(_d(mu), f64p), _p(_d(o), f64p), float(theta), _p(Sh, f64p))
    return Sh.reshape(3, 3)


def cholesky3(S):
    L = np.zeros(9)
    rc = lib().or_cholesky3(_p(_d(S), f64p), _p(L, f64p))
    return None if rc else L.reshape(3, 3)


def lower_inverse3(L):
    M = np.zeros(9)
    lib().or_lower_inverse3(_p(_d(L), f64p), _p(M, f64p))
    return M.reshape(3, 3)


def sigma_points_sqrt(mu, Lsq, ut=None):
    pts, wm, wc = np.zeros(21), np.zeros(7), np.zeros(7)
    rc = lib().or_sigma_points_sqrt(_p(_d(mu), f64p), _p(_d(Lsq), f64p), _p(_ut(ut), f64p), _p(pts, f64p),
                                    _p(wm, f64p), _p(wc, f64p))
    assert rc == 0
    return pts.reshape(7, 3), wm, wc


def ut_affine(mu, q, s, A, b, ut=None):
    mean, cov = np.zeros(2), np.zeros(3)
    lib().or_ut_affine(_p(_d(mu), f64p), _p(_d(q), f64p), _p(_d(s), f64p), _p(_ut(ut), f64p), _p(_d(A), f64p),
                       _p(_d(b), f64p), _p(mean, f64p), _p(cov, f64p))
    return mean, np.array([[cov[0], cov[1]], [cov[1], cov[2]]])


def pose_at(p0, p1, s):
    R, t = np.zeros(9), np.zeros(3)
    lib().or_pose_at(_p(_d(p0), f64p), _p(_d(p1), f64p), float(s), _p(R, f64p), _p(t, f64p))
    return R.reshape(3, 3), t


def lidar_point(x, cfg, p0, p1, K):
    out = np.zeros(4)
    L = make_lidar(cfg)
    lib().or_lidar_point(_p(_d(x), f64p), C.byref(L), _p(_d(p0), f64p), _p(_d(p1), f64p), int(K), _p(out, f64p))
    return out


def camera_point(x, cam, p0, p1, K):
    out = np.zeros(4)
    Cm = make_camera(cam)
    v = lib().or_camera_point(_p(_d(x), f64p), C.byref(Cm), _p(_d(p0), f64p), _p(_d(p1), f64p), int(K),
                              _p(out, f64p))
    return bool(v), out


def camera_unproject(cam, u, v):
    d = np.zeros(3)
    Cm = make_camera(cam)
    ok = lib().or_camera_unproject(C.byref(Cm), float(u), float(v), _p(d, f64p))
    return bool(ok), d


def sh_eval(sh, direction, degree=3):
    out = np.zeros(3)
    lib().or_sh_eval(_p(_d(sh).reshape(-1), f64p), int(degree), _p(_d(direction), f64p), _p(out, f64p))
    return out


def response(mu, Mrows, o, d):
    out = np.zeros(2)
    lib().or_response(_p(_d(mu), f64p), _p(_d(Mrows).reshape(-1), f64p), _p(_d(o), f64p), _p(_d(d), f64p),
                      _p(out, f64p))
    return out[0], out[1]


def sat_query(sat, r_lo, r_hi, c_lo, c_hi):
    sat = np.ascontiguousarray(sat, np.int32)
    return int(lib().or_sat_query(_p(sat, i32p), sat.shape[1], r_lo, r_hi, c_lo, c_hi))
