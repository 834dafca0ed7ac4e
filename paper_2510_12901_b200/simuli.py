"""Thin Python binding of libsimuli (include/simuli.h): argument marshalling only.

Every step of the path runs in libsimuli's CUDA kernels; PyTorch only provides device
memory and streams.  There is no CPU fallback: if libsimuli.so is missing or no CUDA
device is present, calls raise.

The five ABI calls keep their names: ``simuli_build_tiles``, ``simuli_project``,
``simuli_bin_sort``, ``simuli_render_lidar``, ``simuli_render_camera``.  ``LidarRenderer``
and ``CameraRenderer`` hold the device buffers of one sensor + scene and enqueue the three
stages of a frame.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsimuli.so")

SIMULI_OK, SIMULI_ERR_INVALID_ARGUMENT, SIMULI_ERR_CAPACITY, SIMULI_ERR_CUDA, SIMULI_ERR_UNSUPPORTED = range(5)
SENSOR_LIDAR, SENSOR_CAMERA = 0, 1
CAM_PINHOLE_RADTAN, CAM_FISHEYE_KB = 0, 1
RECORD_FLOATS = 20

ABI_VERSION = 12  # include/simuli.h SIMULI_ABI_VERSION
EXPORTED = ["simuli_last_error", "simuli_abi_version", "simuli_build_tiles", "simuli_project",
            "simuli_bin_sort_workspace_size", "simuli_bin_sort", "simuli_render_lidar", "simuli_render_camera",
            "simuli_compose_camera", "simuli_backward_workspace_size", "simuli_backward_lidar",
            "simuli_backward_camera"]

f32p, i32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_int32), C.POINTER(C.c_double)


class SimuliError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libsimuli error {code}: {msg}")
        self.code = code


# ------------------------------------------------------------------------------ structs
class Pose(C.Structure):
    _fields_ = [("q", C.c_float * 4), ("t", C.c_float * 3)]


class Lidar(C.Structure):
    _fields_ = [("n_beams", C.c_int32), ("beam_elevation_rad", f32p), ("n_azimuth", C.c_int32),
                ("azimuth_start_rad", C.c_float), ("spin_direction", C.c_int32), ("min_range_m", C.c_float),
                ("beam_divergence_rad", C.c_float)]


class TilingParams(C.Structure):
    _fields_ = [("n_phi", C.c_int32), ("max_rays_per_tile", C.c_int32), ("hist_bins", C.c_int32),
                ("cull_az_cells", C.c_int32), ("cull_rows_per_tile", C.c_int32)]


_TILING_SCALARS = [("n_phi", C.c_int32), ("n_theta", C.c_int32), ("n_tiles", C.c_int32),
                   ("max_rays_in_tile", C.c_int32), ("sat_rows", C.c_int32), ("sat_cols", C.c_int32),
                   ("n_rays", C.c_int32), ("n_beams", C.c_int32), ("n_azimuth", C.c_int32),
                   ("max_beams_per_elev_tile", C.c_int32), ("max_cols_per_az_tile", C.c_int32),
                   ("pi_f", C.c_float), ("two_pi_f", C.c_float), ("az_tile_scale", C.c_float),
                   ("az_cell_scale", C.c_float)]
_TILING_ARRAYS = [("elev_bounds", f32p), ("cull_row_scale", f32p), ("ray_az", f32p), ("ray_el", f32p),
                  ("ray_s", f32p), ("ray_tile", i32p), ("tile_ray_offsets", i32p), ("tile_rays", i32p),
                  ("sat", i32p), ("elev_tile_beam_offsets", i32p), ("elev_tile_beams", i32p),
                  ("az_tile_col_offsets", i32p), ("az_tile_cols", i32p), ("beam_el_sorted", f32p),
                  ("col_az_sorted", f32p)]


class Tiling(C.Structure):
    _fields_ = _TILING_SCALARS + _TILING_ARRAYS


class TilingDev(C.Structure):
    _fields_ = [("n_phi", C.c_int32), ("n_theta", C.c_int32), ("n_tiles", C.c_int32),
                ("max_rays_in_tile", C.c_int32), ("sat_rows", C.c_int32), ("sat_cols", C.c_int32),
                ("cull_az_cells", C.c_int32), ("cull_rows_per_tile", C.c_int32), ("n_rays", C.c_int32),
                ("n_beams", C.c_int32), ("n_azimuth", C.c_int32), ("max_beams_per_elev_tile", C.c_int32),
                ("max_cols_per_az_tile", C.c_int32), ("pi_f", C.c_float), ("two_pi_f", C.c_float),
                ("az_tile_scale", C.c_float), ("az_cell_scale", C.c_float)] + \
               [(name, C.c_void_p) for name, _ in _TILING_ARRAYS]


class Gaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("quats", C.c_void_p), ("scales", C.c_void_p),
                ("opacity", C.c_void_p), ("sh", C.c_void_p), ("sh_degree", C.c_int32),
                ("actor_id", C.c_void_p), ("actor_pose", C.c_void_p), ("n_actors", C.c_int32)]


class LidarGradIn(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("zeta", "opacity", "depth_accum", "depth", "intensity", "raydrop",
                                          "fwd_zeta", "fwd_opacity", "fwd_depth_accum")]


class CameraGradIn(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("rgb", "opacity", "depth_accum", "depth", "fwd_rgb", "fwd_opacity",
                                          "fwd_depth_accum")]


class GaussianGrads(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("means", "quats", "scales", "opacity", "sh", "actor_pose")]


class CameraCompose(C.Structure):
    _fields_ = [("env_map", C.c_void_p), ("env_h", C.c_int32), ("env_w", C.c_int32), ("grid", C.c_void_p),
                ("grid_h", C.c_int32), ("grid_w", C.c_int32), ("grid_d", C.c_int32)]


class Camera(C.Structure):
    _fields_ = [("model", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float),
                ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("k", C.c_float * 5),
                ("rolling_shutter", C.c_int32), ("near_m", C.c_float), ("max_theta_rad", C.c_float),
                ("tile_px", C.c_int32)]


class ProjectParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lidar", C.POINTER(Lidar)), ("tiling", C.POINTER(TilingDev)),
                ("camera", C.POINTER(Camera)), ("pose_start", Pose), ("pose_end", Pose),
                ("rs_iterations", C.c_int32), ("ut_alpha", C.c_float), ("ut_beta", C.c_float),
                ("ut_kappa", C.c_float), ("extent_sigma", C.c_float), ("enable_culling", C.c_int32),
                ("write_all_records", C.c_int32)]


class Projected(C.Structure):
    _fields_ = [("record", C.c_void_p), ("tile_rect", C.c_void_p), ("depth_key", C.c_void_p),
                ("tile_count", C.c_void_p), ("view_dir", C.c_void_p)]


class RenderParams(C.Structure):
    _fields_ = [("alpha_min", C.c_float), ("alpha_max", C.c_float), ("T_min", C.c_float), ("sh", C.c_void_p),
                ("sh_degree", C.c_int32), ("lidar_producers", C.c_int32)]


class LidarOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("zeta", "opacity", "depth_accum", "depth", "intensity", "raydrop",
                                          "final_T", "n_contrib", "ray_od", "n_visited", "n_inbox")]


class CameraOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("rgb", "opacity", "depth_accum", "depth", "final_T", "n_contrib",
                                          "ray_od", "n_visited", "n_inbox")]


_lib = None


def load():
    """Load libsimuli.so (built in-tree by paper_2510_12901_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libsimuli.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    L.simuli_last_error.restype = C.c_char_p
    L.simuli_abi_version.restype = C.c_int32
    if L.simuli_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libsimuli.so ABI {L.simuli_abi_version()} != binding {ABI_VERSION}; rebuild it")
    L.simuli_build_tiles.argtypes = [C.POINTER(Lidar), C.POINTER(TilingParams), C.POINTER(Tiling)]
    L.simuli_project.argtypes = [C.POINTER(Gaussians), C.POINTER(ProjectParams), C.POINTER(Projected), C.c_void_p]
    L.simuli_bin_sort_workspace_size.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]
    L.simuli_bin_sort.argtypes = [C.POINTER(Projected), C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
                                  C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
    L.simuli_render_lidar.argtypes = [C.POINTER(Projected), C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(ProjectParams), C.POINTER(RenderParams), C.POINTER(LidarOut),
                                      C.c_void_p]
    L.simuli_render_camera.argtypes = [C.POINTER(Projected), C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.POINTER(ProjectParams), C.POINTER(RenderParams), C.POINTER(CameraOut),
                                       C.c_void_p]
    L.simuli_backward_workspace_size.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]
    for nm, gin in (("simuli_backward_lidar", LidarGradIn), ("simuli_backward_camera", CameraGradIn)):
        getattr(L, nm).argtypes = [C.POINTER(Gaussians), C.POINTER(Projected), C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(ProjectParams), C.POINTER(RenderParams), C.POINTER(gin),
                                   C.POINTER(GaussianGrads), C.c_void_p, C.c_size_t, C.c_void_p]
    L.simuli_compose_camera.argtypes = [C.POINTER(ProjectParams), C.POINTER(CameraCompose), C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
    for name in EXPORTED:
        if name not in ("simuli_last_error", "simuli_abi_version"):
            getattr(L, name).restype = C.c_int32
    _lib = L
    return L


def _check(code):
    if code != SIMULI_OK:
        raise SimuliError(code, load().simuli_last_error().decode())


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_pose(p) -> Pose:
    q = np.asarray(p["q"], np.float32)
    t = np.asarray(p["t"], np.float32)
    return Pose((C.c_float * 4)(*q.tolist()), (C.c_float * 3)(*t.tolist()))


# ------------------------------------------------------------------------------ ABI calls
def simuli_build_tiles(cfg) -> dict:
    """Host call: Proc. ElevationTiling + ray table + SAT for a LidarConfig (synth)."""
    L = load()
    beams = np.ascontiguousarray(cfg.beams, np.float32)
    lid = Lidar(int(beams.shape[0]), beams.ctypes.data_as(f32p), int(cfg.n_azimuth), float(cfg.azimuth_start),
                int(cfg.spin_direction), float(cfg.min_range))
    prm = TilingParams(cfg.n_phi, cfg.max_rays_per_tile, cfg.hist_bins, cfg.cull_az_cells, cfg.cull_rows_per_tile)
    t = Tiling()
    _check(L.simuli_build_tiles(C.byref(lid), C.byref(prm), C.byref(t)))
    sizes = {"elev_bounds": (t.n_phi + 1, np.float32), "cull_row_scale": (t.n_phi, np.float32),
             "ray_az": (t.n_rays, np.float32), "ray_el": (t.n_rays, np.float32), "ray_s": (t.n_rays, np.float32),
             "ray_tile": (t.n_rays, np.int32), "tile_ray_offsets": (t.n_tiles + 1, np.int32),
             "tile_rays": (t.n_rays, np.int32), "sat": (t.sat_rows * t.sat_cols, np.int32),
             "elev_tile_beam_offsets": (t.n_phi + 1, np.int32), "elev_tile_beams": (t.n_beams, np.int32),
             "az_tile_col_offsets": (t.n_theta + 1, np.int32), "az_tile_cols": (t.n_azimuth, np.int32),
             "beam_el_sorted": (t.n_beams, np.float32), "col_az_sorted": (t.n_azimuth, np.float32)}
    arrays = {k: np.zeros(n, dt) for k, (n, dt) in sizes.items()}
    for k, a in arrays.items():
        setattr(t, k, a.ctypes.data_as(f32p if a.dtype == np.float32 else i32p))
    _check(L.simuli_build_tiles(C.byref(lid), C.byref(prm), C.byref(t)))
    out = {name: getattr(t, name) for name, _ in _TILING_SCALARS}
    out.update(arrays)
    out["sat"] = arrays["sat"].reshape(t.sat_rows, t.sat_cols)
    out["cull_az_cells"] = cfg.cull_az_cells
    out["cull_rows_per_tile"] = cfg.cull_rows_per_tile
    return out


def simuli_project(gaussians: Gaussians, params: ProjectParams, out: Projected, stream=None):
    _check(load().simuli_project(C.byref(gaussians), C.byref(params), C.byref(out), _stream(stream)))


def simuli_bin_sort_workspace_size(n, capacity, n_tiles) -> int:
    b = C.c_size_t(0)
    _check(load().simuli_bin_sort_workspace_size(int(n), int(capacity), int(n_tiles), C.byref(b)))
    return int(b.value)


def simuli_bin_sort(proj: Projected, n, n_tiles, n_cols_total, workspace, capacity, sorted_keys, sorted_ids,
                    tile_ranges, n_pairs_dev, stream=None, tile_order=None, n_pairs_max=None) -> int | None:
    req = C.c_int64(-1)
    code = load().simuli_bin_sort(C.byref(proj), int(n), int(n_tiles), int(n_cols_total), _ptr(workspace),
                                  workspace.numel() * workspace.element_size(), int(capacity), _ptr(sorted_keys),
                                  _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order), _ptr(n_pairs_dev),
                                  _ptr(n_pairs_max), C.byref(req),
                                  _stream(stream))
    if code == SIMULI_ERR_CAPACITY:
        return int(req.value)
    _check(code)
    return None


def simuli_render_lidar(proj, sorted_ids, tile_ranges, params, rparams, out: LidarOut, stream=None, tile_order=None):
    _check(load().simuli_render_lidar(C.byref(proj), _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order),
                                      C.byref(params),
                                      C.byref(rparams), C.byref(out), _stream(stream)))


def simuli_compose_camera(params, env, grid, rgb_fg, opacity, rgb_out, stream=None):
    """Eq. 2 (env map + bilateral grid); env [He, We, 3] / grid [gd, gh, gw, 12] device float32 or None."""
    comp = CameraCompose(None if env is None else env.data_ptr(), 0 if env is None else env.shape[0],
                         0 if env is None else env.shape[1], None if grid is None else grid.data_ptr(),
                         0 if grid is None else grid.shape[1], 0 if grid is None else grid.shape[2],
                         0 if grid is None else grid.shape[0])
    _check(load().simuli_compose_camera(C.byref(params), C.byref(comp), _ptr(rgb_fg), _ptr(opacity), _ptr(rgb_out),
                                        _stream(stream)))


def simuli_backward_workspace_size(n, pair_capacity=0, n_tiles=0):
    b = C.c_size_t(0)
    _check(load().simuli_backward_workspace_size(int(n), int(pair_capacity), int(n_tiles), C.byref(b)))
    return int(b.value)


def _grad_structs(frame, grads, names, gin_cls, fwd):
    import torch
    sc = frame.scene
    keys = ("means", "quats", "scales", "opacity", "sh") + (("actor_pose",) if sc.get("actor_pose") is not None else ())
    out = {k: torch.empty_like(sc[k]) for k in keys}  # with a scene graph: object-frame and pose gradients
    gin = gin_cls(*[_ptr(grads.get(k)) if grads.get(k) is not None else None for k in names],
                  *[_ptr(t) if t is not None else None for t in fwd])
    gout = GaussianGrads(*[_ptr(out[k]) for k in keys])
    return out, gin, gout


def simuli_backward(frame, grads, stream=None, use_forward_totals=True):
    """Backward of the frame's last forward (A31): grads = upstream gradients by output
    name (device float32; missing = 0).  Returns the particle parameter gradients.
    use_forward_totals: pass the forward's zeta / opacity / depth_accum outputs so the
    backward skips its totals pass."""
    lidar = isinstance(frame, LidarRenderer)
    names = ("zeta", "opacity", "depth_accum", "depth", "intensity", "raydrop") if lidar else \
        ("rgb", "opacity", "depth_accum", "depth")
    grads = {k: v.contiguous() for k, v in grads.items() if v is not None}
    fk = ("zeta" if lidar else "rgb", "opacity", "depth_accum")
    fwd = [frame.out.get(k) for k in fk] if use_forward_totals else [None, None, None]
    if any(t is None for t in fwd):
        fwd = [None, None, None]
    out, gin, gout = _grad_structs(frame, grads, names, LidarGradIn if lidar else CameraGradIn, fwd)
    ws = frame._bwd_workspace()
    frame._on_stream(stream, ws, *out.values())
    fn = load().simuli_backward_lidar if lidar else load().simuli_backward_camera
    _check(fn(C.byref(frame.gauss), C.byref(frame.projected), _ptr(frame.sorted_ids), _ptr(frame.tile_ranges),
              _ptr(frame.tile_order), C.byref(frame.params), C.byref(frame.rparams), C.byref(gin), C.byref(gout), _ptr(ws), ws.numel(),
              _stream(stream)))
    frame._keep_grads = grads  # alive until the enqueued work has run
    return out


def simuli_render_camera(proj, sorted_ids, tile_ranges, params, rparams, out: CameraOut, stream=None,
                         tile_order=None):
    _check(load().simuli_render_camera(C.byref(proj), _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order),
                                       C.byref(params),
                                       C.byref(rparams), C.byref(out), _stream(stream)))


# ------------------------------------------------------------------------------ helpers
def to_device_scene(scene: dict, device="cuda"):
    """Upload a synth scene (float32 numpy) to device tensors; optional scene-graph keys
    actor_id [n] int32 and actor_pose [n_actors, 7] float32 (q w,x,y,z, t) (A29)."""
    import torch
    out = {k: torch.from_numpy(np.ascontiguousarray(scene[k], np.float32)).to(device)
           for k in ("means", "quats", "scales", "opacity", "sh")}
    if scene.get("actor_id") is not None:
        out["actor_id"] = torch.from_numpy(np.ascontiguousarray(scene["actor_id"], np.int32)).to(device)
        out["actor_pose"] = torch.from_numpy(np.ascontiguousarray(scene["actor_pose"], np.float32)).to(device)
    return out


def gaussians_struct(scene_dev) -> Gaussians:
    n = int(scene_dev["means"].shape[0])
    sh = scene_dev["sh"]
    ncoef = sh.numel() // max(n, 1) // 3 if n else 16
    deg = {1: 0, 4: 1, 9: 2, 16: 3}[ncoef]
    act = scene_dev.get("actor_id")
    return Gaussians(n, _ptr(scene_dev["means"]), _ptr(scene_dev["quats"]), _ptr(scene_dev["scales"]),
                     _ptr(scene_dev["opacity"]), _ptr(sh), deg, _ptr(act),
                     _ptr(scene_dev["actor_pose"] if act is not None else None),
                     int(scene_dev["actor_pose"].shape[0]) if act is not None else 0)


class _Frame:
    """Common device buffers of one sensor frame (projection + binning)."""

    def _alloc_common(self, n, n_tiles, capacity):
        import torch
        dev = self.device
        self.n = n
        self.record = torch.empty((max(n, 1), RECORD_FLOATS), dtype=torch.float32, device=dev)
        self.tile_rect = torch.empty((max(n, 1), 4), dtype=torch.int32, device=dev)
        self.depth_key = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        self.tile_count = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.tile_ranges = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
        self.tile_order = torch.empty(n_tiles, dtype=torch.int32, device=dev)
        self.n_pairs = torch.zeros(1, dtype=torch.int64, device=dev)
        # running maximum of the pair count over asynchronous bin_sort calls (device-side,
        # updated on the call's stream); check_capacity() compares it with the capacity
        self.max_pairs = torch.zeros(1, dtype=torch.int64, device=dev)
        self.projected = Projected(_ptr(self.record), _ptr(self.tile_rect), _ptr(self.depth_key),
                                   _ptr(self.tile_count))
        self.set_capacity(capacity)

    def set_capacity(self, capacity):
        import torch
        capacity = max(int(capacity), 1)
        self.capacity = capacity
        self.sorted_keys = torch.empty(capacity, dtype=torch.int64, device=self.device)
        self.sorted_ids = torch.empty(capacity, dtype=torch.int32, device=self.device)
        ws = simuli_bin_sort_workspace_size(self.n, capacity, self.n_tiles)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
        if getattr(self, "max_pairs", None) is not None:
            self.max_pairs.zero_()

    def _on_stream(self, stream, *tensors):
        """Tensors allocated on the current torch stream but used by kernels enqueued on
        `stream`: tell the caching allocator (record_stream) so their memory is not reused
        by current-stream work before `stream` has finished with it."""
        if stream is None:
            return
        import torch
        st = stream if isinstance(stream, torch.cuda.Stream) else None
        if st is None or st == torch.cuda.current_stream(self.device):
            return
        for t in tensors:
            if t is not None:
                t.record_stream(st)

    def check_capacity(self):
        """Raise if any asynchronous bin_sort since the last set_capacity() had more pairs
        than the capacity (its tile lists were truncated; simuli.h: simuli_bin_sort).
        Synchronises with the device."""
        mp = int(self.max_pairs.item())
        if mp > self.capacity:
            raise SimuliError(2, f"bin_sort: {mp} pairs exceeded the pair capacity {self.capacity}: outputs of "
                                 f"that frame are incomplete; call set_capacity() or bin_sort(sync_capacity=True)")
        return mp

    def project(self, stream=None):
        simuli_project(self.gauss, self.params, self.projected, stream)

    def requires_grad(self, flag=True):
        """Write the per-particle SH view directions the backward needs (A31)."""
        import torch
        self.view_dir = torch.zeros((max(self.n, 1), 3), dtype=torch.float32, device=self.device) if flag else None
        self.projected.view_dir = _ptr(self.view_dir).value if flag else None

    def _bwd_workspace(self):
        import torch
        need = simuli_backward_workspace_size(self.n, self.capacity, self.n_tiles)
        if getattr(self, "_bws", None) is None or self._bws.numel() < need:
            self._bws = torch.empty(max(need, 16), dtype=torch.uint8, device=self.device)
        return self._bws

    def backward(self, grads, stream=None, use_forward_totals=True):
        """Gradients of the particle parameters from upstream output gradients (A31).
        Checks first that no asynchronous bin_sort overflowed its pair capacity (one
        device sync): gradients of a truncated forward would be silently wrong."""
        self.check_capacity()
        return simuli_backward(self, grads, stream, use_forward_totals)

    keep_keys = True  # also write the u64 (tile | depth) keys (tests); the renderer needs only ids

    def bin_sort(self, stream=None, sync_capacity=False):
        """Duplicate + sort.  sync_capacity=True: one host sync to grow buffers if needed."""
        cap = -self.capacity if sync_capacity else self.capacity
        keys = self.sorted_keys if self.keep_keys else None
        # asynchronous calls raise the sticky device-side maximum checked by check_capacity()
        need = simuli_bin_sort(self.projected, self.n, self.n_tiles, self.n_cols_total, self.workspace, cap,
                               keys, self.sorted_ids, self.tile_ranges, self.n_pairs, stream,
                               self.tile_order, None if sync_capacity else self.max_pairs)
        if need is not None:
            self.set_capacity(int(need * 1.25) + 1024)
            keys = self.sorted_keys if self.keep_keys else None
            need = simuli_bin_sort(self.projected, self.n, self.n_tiles, self.n_cols_total, self.workspace,
                                   -self.capacity, keys, self.sorted_ids, self.tile_ranges,
                                   self.n_pairs, stream, self.tile_order)
            assert need is None
        self._on_stream(stream, self.sorted_keys, self.sorted_ids, self.workspace)

    def set_poses(self, pose_start, pose_end):
        self.params.pose_start = make_pose(pose_start)
        self.params.pose_end = make_pose(pose_end)


class LidarRenderer(_Frame):
    """One spinning LiDAR + one Gaussian set G_l resident on the device.

    enable_culling: 0 off, 1 the paper's dense-grid SAT culling (Proc. RayOccupancyCount /
    ProjectParticles), 2 exact ray containment per render tile (A32, default); the rendered
    outputs are identical in all three modes, only the tile lists differ."""

    def __init__(self, cfg, scene_dev, capacity=None, device="cuda", enable_culling=2, write_all_records=False,
                 ut=(1.0, 2.0, 0.0), extent_sigma=3.0, render_params=(1.0 / 255.0, 0.99, 1e-4), per_ray_sh=False,
                 render_producers=0):
        import torch
        self.device = device
        self.cfg = cfg
        self.scene = scene_dev
        self.gauss = gaussians_struct(scene_dev)
        self.tiling_host = simuli_build_tiles(cfg)
        th = self.tiling_host
        self.tiling_dev_tensors = {}
        for name, _ in _TILING_ARRAYS:
            a = th[name].reshape(-1)
            self.tiling_dev_tensors[name] = torch.from_numpy(a.copy()).to(device)
        td = TilingDev(th["n_phi"], th["n_theta"], th["n_tiles"], th["max_rays_in_tile"], th["sat_rows"],
                       th["sat_cols"], cfg.cull_az_cells, cfg.cull_rows_per_tile, th["n_rays"], th["n_beams"],
                       th["n_azimuth"], th["max_beams_per_elev_tile"], th["max_cols_per_az_tile"], th["pi_f"], th["two_pi_f"], th["az_tile_scale"], th["az_cell_scale"],
                       *[self.tiling_dev_tensors[name].data_ptr() for name, _ in _TILING_ARRAYS])
        self.tiling_dev = td
        beams = np.ascontiguousarray(cfg.beams, np.float32)
        self._beams = beams
        self.lidar = Lidar(int(beams.shape[0]), beams.ctypes.data_as(f32p), int(cfg.n_azimuth),
                           float(cfg.azimuth_start), int(cfg.spin_direction), float(cfg.min_range),
                           float(getattr(cfg, "beam_divergence", 0.0)))
        self.params = ProjectParams(SENSOR_LIDAR, C.pointer(self.lidar), C.pointer(self.tiling_dev), None,
                                    make_pose(cfg.pose_start), make_pose(cfg.pose_end), int(cfg.rs_iterations),
                                    ut[0], ut[1], ut[2], extent_sigma, int(enable_culling), int(write_all_records))
        self.rparams = RenderParams(*render_params, None, 0)
        # render pipeline shape (simuli.h): 0 = hybrid default, 1..3 = producer / consumer
        # with that many producers (3 = latency), 4 = one warp per item; identical outputs
        self.rparams.lidar_producers = int(render_producers)
        if per_ray_sh:  # Eq. 1 literally: SH_i(d) per (ray, particle) (A30)
            self.rparams.sh = scene_dev["sh"].data_ptr()
            self.rparams.sh_degree = self.gauss.sh_degree
        self.n_tiles = th["n_tiles"]
        self.n_cols_total = th["n_theta"]
        self.n_rays = th["n_rays"]
        n = int(scene_dev["means"].shape[0])
        self._alloc_common(n, self.n_tiles, capacity if capacity is not None else max(4 * n, 1024))
        R = self.n_rays
        f = lambda *s: torch.empty(s, dtype=torch.float32, device=device)  # noqa: E731
        self.out = {"zeta": f(R, 3), "opacity": f(R), "depth_accum": f(R), "depth": f(R), "intensity": f(R),
                    "raydrop": f(R), "final_T": f(R), "n_contrib": torch.empty(R, dtype=torch.int32, device=device),
                    "ray_od": None, "n_visited": None, "n_inbox": None}
        self._out_struct()

    def _out_struct(self):
        o = self.out
        self.out_struct = LidarOut(*[_ptr(o[k]) for k in ("zeta", "opacity", "depth_accum", "depth", "intensity",
                                                          "raydrop", "final_T", "n_contrib", "ray_od", "n_visited",
                                                          "n_inbox")])

    def want_counters(self, flag=True):
        import torch
        for k in ("n_visited", "n_inbox"):
            self.out[k] = torch.empty(self.n_rays, dtype=torch.int32, device=self.device) if flag else None
        self._out_struct()

    def want_ray_od(self, flag=True):
        import torch
        self.out["ray_od"] = torch.empty((self.n_rays, 6), dtype=torch.float64, device=self.device) if flag else None
        self._out_struct()

    def render(self, stream=None):
        simuli_render_lidar(self.projected, self.sorted_ids, self.tile_ranges, self.params, self.rparams,
                            self.out_struct, stream, self.tile_order)

    def scan(self, pose_start=None, pose_end=None, stream=None, sync_capacity=False):
        """Enqueue one full scan: project -> bin_sort -> render (north-star stages 1, 3-5)."""
        if pose_start is not None:
            self.set_poses(pose_start, pose_end if pose_end is not None else pose_start)
        self.project(stream)
        self.bin_sort(stream, sync_capacity)
        self.render(stream)
        return self.out


class CameraRenderer(_Frame):
    """One distorted rolling-shutter camera + one Gaussian set G_c resident on the device."""

    def __init__(self, cam, scene_dev, capacity=None, device="cuda", write_all_records=False, ut=(1.0, 2.0, 0.0),
                 extent_sigma=3.0, render_params=(1.0 / 255.0, 0.99, 1e-4), per_ray_sh=False):
        import torch
        self.device = device
        self.cam_cfg = cam
        self.scene = scene_dev
        self.gauss = gaussians_struct(scene_dev)
        self.camera = Camera(int(cam.model), int(cam.width), int(cam.height), float(cam.fx), float(cam.fy),
                             float(cam.cx), float(cam.cy), (C.c_float * 5)(*[float(x) for x in cam.k]),
                             int(cam.rolling_shutter), float(cam.near), float(cam.max_theta), int(cam.tile_px))
        self.params = ProjectParams(SENSOR_CAMERA, None, None, C.pointer(self.camera), make_pose(cam.pose_start),
                                    make_pose(cam.pose_end), int(cam.rs_iterations), ut[0], ut[1], ut[2],
                                    extent_sigma, 0, int(write_all_records))
        self.rparams = RenderParams(*render_params, None, 0)
        if per_ray_sh:  # Eq. 1 literally: SH_i(d) per (ray, particle) (A30)
            self.rparams.sh = scene_dev["sh"].data_ptr()
            self.rparams.sh_degree = self.gauss.sh_degree
        tp = cam.tile_px
        self.Wt, self.Ht = (cam.width + tp - 1) // tp, (cam.height + tp - 1) // tp
        self.n_tiles = self.Wt * self.Ht
        self.n_cols_total = self.Wt
        n = int(scene_dev["means"].shape[0])
        self._alloc_common(n, self.n_tiles, capacity if capacity is not None else max(8 * n, 1024))
        P = cam.width * cam.height
        f = lambda *s: torch.empty(s, dtype=torch.float32, device=device)  # noqa: E731
        self.out = {"rgb": f(P, 3), "opacity": f(P), "depth_accum": f(P), "depth": f(P), "final_T": f(P),
                    "n_contrib": torch.empty(P, dtype=torch.int32, device=device), "ray_od": None,
                    "n_visited": None, "n_inbox": None}
        self._out_struct()

    def _out_struct(self):
        o = self.out
        self.out_struct = CameraOut(*[_ptr(o[k]) for k in ("rgb", "opacity", "depth_accum", "depth", "final_T",
                                                           "n_contrib", "ray_od", "n_visited", "n_inbox")])

    def want_counters(self, flag=True):
        import torch
        P = self.cam_cfg.width * self.cam_cfg.height
        for k in ("n_visited", "n_inbox"):
            self.out[k] = torch.empty(P, dtype=torch.int32, device=self.device) if flag else None
        self._out_struct()

    def want_ray_od(self, flag=True):
        import torch
        P = self.cam_cfg.width * self.cam_cfg.height
        self.out["ray_od"] = torch.empty((P, 6), dtype=torch.float64, device=self.device) if flag else None
        self._out_struct()

    def render(self, stream=None):
        simuli_render_camera(self.projected, self.sorted_ids, self.tile_ranges, self.params, self.rparams,
                             self.out_struct, stream, self.tile_order)

    def compose(self, env=None, grid=None, stream=None):
        """Eq. 2 final colour from the last frame's c_f and omega (env map, bilateral grid)."""
        import torch
        out = torch.empty_like(self.out["rgb"])
        simuli_compose_camera(self.params, env, grid, self.out["rgb"], self.out["opacity"], out, stream)
        return out

    def frame(self, pose_start=None, pose_end=None, stream=None, sync_capacity=False):
        if pose_start is not None:
            self.set_poses(pose_start, pose_end if pose_end is not None else pose_start)
        self.project(stream)
        self.bin_sort(stream, sync_capacity)
        self.render(stream)
        return self.out
