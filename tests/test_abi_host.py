"""C-ABI library checks that need no GPU (-m "not gpu"): the library loads, exports every
symbol include/simuli.h declares, and the host-side simuli_build_tiles (Proc.
ElevationTiling + ray table + SAT) is bit-exact against the oracle."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2510_12901_b200 import synth as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_12901_b200 import build as B
    B.build()
    from paper_2510_12901_b200 import simuli as SM
    return SM


def header_symbols():
    src = open(os.path.join(ROOT, "include", "simuli.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(simuli_\w+)\s*\(", src, re.M)))


def test_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert set(syms) >= {"simuli_build_tiles", "simuli_project", "simuli_bin_sort", "simuli_render_lidar",
                         "simuli_render_camera"}
    L = lib.load()
    for s in syms:
        assert hasattr(L, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    assert set(syms) <= exported
    assert set(lib.EXPORTED) == set(syms)
    assert L.simuli_abi_version() == 12


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _compare_tiling(cfg, SM, O):
    p = SM.simuli_build_tiles(cfg)
    o = O.Tiling(cfg)
    assert (p["n_phi"], p["n_theta"], p["n_tiles"], p["max_rays_in_tile"]) == (o.n_phi, o.n_theta, o.n_tiles,
                                                                              o.max_rays_in_tile)
    assert (p["sat_rows"], p["sat_cols"]) == (o.sat_rows, o.sat_cols)
    for k in ("pi_f", "two_pi_f", "az_tile_scale", "az_cell_scale"):
        assert np.float32(p[k]).view(np.uint32) == np.float32(getattr(o, k)).view(np.uint32), k
    pairs = [("elev_bounds", o.bounds), ("cull_row_scale", o.cull_row_scale), ("ray_az", o.ray_az),
             ("ray_el", o.ray_el), ("ray_s", o.ray_s), ("ray_tile", o.ray_tile),
             ("tile_ray_offsets", o.tile_ray_offsets), ("tile_rays", o.tile_rays), ("sat", o.sat)]
    for name, ref in pairs:
        a = np.asarray(p[name])
        assert a.shape == ref.shape, name
        assert np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a,
                              ref.view(np.uint32) if ref.dtype == np.float32 else ref), name
    # beam / column CSR consistent with the ray table
    B, A = p["n_beams"], p["n_azimuth"]
    for e in range(p["n_phi"]):
        for b in p["elev_tile_beams"][p["elev_tile_beam_offsets"][e]:p["elev_tile_beam_offsets"][e + 1]]:
            assert p["ray_tile"][b * A] // p["n_theta"] == e
    for c in range(p["n_theta"]):
        for j in p["az_tile_cols"][p["az_tile_col_offsets"][c]:p["az_tile_col_offsets"][c + 1]]:
            assert p["ray_tile"][j] % p["n_theta"] == c
    assert p["elev_tile_beam_offsets"][-1] == B and p["az_tile_col_offsets"][-1] == A
    assert p["max_beams_per_elev_tile"] == np.diff(p["elev_tile_beam_offsets"]).max()
    assert p["max_cols_per_az_tile"] == np.diff(p["az_tile_col_offsets"]).max()
    # exact culling's search arrays (A32): the beam elevations / column azimuths, ascending
    A = p["n_azimuth"]
    assert np.array_equal(p["beam_el_sorted"], np.sort(p["ray_el"][::A]))
    assert np.array_equal(p["col_az_sorted"], np.sort(p["ray_az"][:A]))


@pytest.mark.parametrize("name", ["A", "B", "C", "tiny"])
def test_build_tiles_bit_exact_vs_oracle(lib, oracle_mod, name):
    _compare_tiling(S.lidar_config(name), lib, oracle_mod)


def test_build_tiles_random_tables_bit_exact(lib, oracle_mod):
    rng = np.random.default_rng(21)
    for trial in range(60):
        B = int(rng.integers(1, 96))
        beams = rng.uniform(-0.6, 0.4, B).astype(np.float32)
        if trial % 4 == 0:
            beams = np.round(beams, 2).astype(np.float32)
        cfg = S.LidarConfig("r", beams, int(rng.integers(8, 3000)), n_phi=int(rng.integers(1, 70)),
                            max_rays_per_tile=int(rng.choice([8, 16, 32, 64, 128, 256])),
                            cull_az_cells=int(rng.choice([64, 1600])), cull_rows_per_tile=int(rng.choice([4, 8])),
                            azimuth_start=float(np.float32(rng.uniform(-np.pi, np.pi))),
                            spin_direction=int(rng.choice([-1, 1])))
        _compare_tiling(cfg, lib, oracle_mod)


def test_build_tiles_errors(lib):
    cfg = S.lidar_config("A")
    cfg.n_phi = 500  # > hist_bins
    with pytest.raises(lib.SimuliError) as e:
        lib.simuli_build_tiles(cfg)
    assert e.value.code == lib.SIMULI_ERR_INVALID_ARGUMENT and "histogram resolution" in str(e.value)
    cfg = S.lidar_config("A")
    cfg.spin_direction = 2
    with pytest.raises(lib.SimuliError):
        lib.simuli_build_tiles(cfg)
    # all elevations identical -> a single elevation tile, not an error
    cfg = S.LidarConfig("flat", np.zeros(16, np.float32), 100, n_phi=4)
    t = lib.simuli_build_tiles(cfg)
    assert t["n_phi"] == 1 and t["n_theta"] == int(np.ceil(16 * 100 / 32))


def test_workspace_size_and_bad_args(lib):
    assert lib.simuli_bin_sort_workspace_size(1000, 4000, 512) > 4000 * 12
    L = lib.load()
    assert L.simuli_project(None, None, None, None) == lib.SIMULI_ERR_INVALID_ARGUMENT
    assert b"NULL" in L.simuli_last_error()
    assert L.simuli_render_lidar(None, None, None, None, None, None, None, None) == lib.SIMULI_ERR_INVALID_ARGUMENT
    assert L.simuli_render_camera(None, None, None, None, None, None, None, None) == lib.SIMULI_ERR_INVALID_ARGUMENT
    assert L.simuli_compose_camera(None, None, None, None, None, None) == lib.SIMULI_ERR_INVALID_ARGUMENT
    size = ctypes.c_size_t(0)
    assert L.simuli_bin_sort_workspace_size(-1, 10, 1, ctypes.byref(size)) == lib.SIMULI_ERR_INVALID_ARGUMENT
    # backward (A31): size query and argument checks run on the host
    assert L.simuli_backward_workspace_size(1000, 0, 0, ctypes.byref(size)) == lib.SIMULI_OK
    assert 1000 * 64 <= size.value < 1000 * 64 + 8192
    assert L.simuli_backward_workspace_size(1000, 4096, 10, ctypes.byref(size)) == lib.SIMULI_OK
    assert size.value >= 1000 * 64 + (10 + 4) * 8 * 512
    assert L.simuli_backward_workspace_size(-1, 0, 0, ctypes.byref(size)) == lib.SIMULI_ERR_INVALID_ARGUMENT
    for fn in (L.simuli_backward_lidar, L.simuli_backward_camera):
        assert fn(None, None, None, None, None, None, None, None, None, None, 0, None) == lib.SIMULI_ERR_INVALID_ARGUMENT
        assert b"NULL" in L.simuli_last_error()


def test_backward_argument_errors(lib):
    """Host-side checks of simuli_backward_* (no device memory is touched: dummy aligned
    addresses): missing view_dir, a small workspace, per-ray SH of the wrong degree or a
    scene graph without poses -> INVALID_ARGUMENT."""
    C = ctypes
    L = lib.load()
    fake = 1 << 20  # never dereferenced: every check below fails before a launch
    G = lib.Gaussians(10, fake, fake, fake, fake, fake, 3, None, None, 0)
    proj = lib.Projected(fake, fake, fake, fake, None)
    rp = lib.RenderParams(1 / 255, 0.99, 1e-4, None, 0)
    gout = lib.GaussianGrads(fake, fake, fake, fake, fake)
    gin = lib.CameraGradIn()
    cam = lib.Camera(1, 64, 48, 50.0, 50.0, 32.0, 24.0, (C.c_float * 5)(0, 0, 0, 0, 0), 1, 0.05, 1.7, 16)
    P = lib.ProjectParams(lib.SENSOR_CAMERA, None, None, C.pointer(cam), lib.make_pose({"q": [1, 0, 0, 0], "t": [0, 0, 0]}),
                          lib.make_pose({"q": [1, 0, 0, 0], "t": [0, 0, 0]}), 1, 1.0, 2.0, 0.0, 3.0, 0, 0)
    args = lambda ws: (C.byref(G), C.byref(proj), fake, fake, None, C.byref(P), C.byref(rp), C.byref(gin),  # noqa: E731
                       C.byref(gout), fake, ws, None)
    assert L.simuli_backward_camera(*args(640)) == lib.SIMULI_ERR_INVALID_ARGUMENT
    assert b"view_dir" in L.simuli_last_error()
    proj.view_dir = fake
    assert L.simuli_backward_camera(*args(639)) == lib.SIMULI_ERR_INVALID_ARGUMENT  # workspace < 10 x 64 B
    rp.sh = fake  # per-ray SH of another degree than the particles'
    assert L.simuli_backward_camera(*args(640)) == lib.SIMULI_ERR_INVALID_ARGUMENT
    assert b"degree" in L.simuli_last_error()
    rp.sh = None
    G.actor_id, G.actor_pose, G.n_actors = fake, None, 1  # scene graph without poses
    assert L.simuli_backward_camera(*args(640)) == lib.SIMULI_ERR_INVALID_ARGUMENT
