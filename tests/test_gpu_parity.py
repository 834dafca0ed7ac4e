"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the CPU oracle.

Tolerances (BASELINE.json north star): tile boundaries, tile-Gaussian lists and sorted key
order bit-exact; depth within 1e-3 m (rays with omega >= 0.5, A16); intensity, ray drop,
colour and opacity within 1e-4 absolute.  Tier 1 feeds the oracle stage the GPU's
previous-stage outputs (so every discrete decision uses identical float32 values); tier 2
runs the oracle from scratch and excludes the rays it flags as threshold-ambiguous (A23),
which must stay below 0.5 %.
"""
import numpy as np
import pytest

from paper_2510_12901_b200 import synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_FEAT = 1e-4
TOL_DEPTH = 1e-3
# A23 flag margins: box edges (rad / px) at the measured GPU-vs-oracle box error bound
# (LiDAR: sigma point 0 in double, offsets in float32 -> <= 1 float32 ulp at |phi| ~ pi,
# measured max 2.38e-7 rad in azimuth and elevation),
# alpha / T / tau thresholds at the float32 response error; box-edge flips only count when
# the particle's alpha*T could move an output by more than a tenth of the tolerance.
LIDAR_EPS = {"a": 3e-7, "b": 3e-7, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4, "impact": 5e-6}
# camera boxes come from an all-float32 UT (no double sigma point 0): measured max GPU-vs-oracle
# edge error 6.1e-4 px (10 float32 ulps at x ~ 1100 px, a near particle of the 4M config-E scene;
# config D: < 5e-4); margin 1e-3 px
CAMERA_EPS = {"a": 1e-3, "b": 1e-3, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4, "impact": 5e-6, "amb_a": 20.0,
              "amb_b": 20.0}
# share of rays the oracle may flag in tier 2; config B's rays traverse ~360
# list entries each, its flag rate at the margins above is ~0.3 %
FLAG_BUDGET = {"default": 0.005, "B": 0.005}


@pytest.fixture(scope="module")
def SM():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2510_12901_b200 import build as B
    B.build()
    from paper_2510_12901_b200 import simuli
    return simuli


def gpu_records(r):
    """The GPU's 80-byte records as the oracle's record dict.  Rows of particles the GPU did
    not write (tile count 0 without write_all_records: never listed, never read) are set to
    NaN explicitly instead of passing on whatever the buffer held."""
    raw = r.record.cpu().numpy().copy()
    written = r.tile_count.cpu().numpy() > 0
    if r.params.write_all_records:
        written |= np.isfinite(raw[:, 16])
    raw[~written] = np.nan
    rec = raw.astype(np.float64)
    return {"mu": rec[:, 0:3], "Mrows": rec[:, 3:12], "sigma": rec[:, 12], "feat": rec[:, 13:16],
            "box": raw[:, 16:20].copy()}


def lidar_run(SM, cfg, scene, **kw):
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), **kw)
    r.want_ray_od(True)
    r.scan(sync_capacity=True)
    torch.cuda.synchronize()
    return r


def sorted_lists(r):
    P = int(r.n_pairs.item())
    return (r.sorted_keys[:P].cpu().numpy().view(np.uint64), r.sorted_ids[:P].cpu().numpy().view(np.uint32),
            r.tile_ranges.cpu().numpy())


def compare_lidar(out, ref, mask=None, tol=TOL_FEAT):
    g = {k: out[k].cpu().numpy().astype(np.float64) for k in ("opacity", "intensity", "raydrop", "depth")}
    zeta = out["zeta"].cpu().numpy().astype(np.float64)
    m = np.ones(len(g["opacity"]), bool) if mask is None else mask
    errs = {"opacity": np.abs(g["opacity"] - ref["opacity"])[m].max(initial=0),
            "intensity": np.abs(g["intensity"] - ref["intensity"])[m].max(initial=0),
            "raydrop": np.abs(g["raydrop"] - ref["raydrop"])[m].max(initial=0),
            "zeta": np.abs(zeta - ref["feat"])[m].max(initial=0)}
    dm = m & (ref["opacity"] >= 0.5)
    errs["depth"] = np.abs(g["depth"] - ref["depth"])[dm].max(initial=0)
    assert max(errs[k] for k in ("opacity", "intensity", "raydrop", "zeta")) < tol, errs
    assert errs["depth"] < TOL_DEPTH, errs
    return errs


# ------------------------------------------------------------------ stage 1 (a1): projection
@pytest.mark.parametrize("config", ["A", "tiny", "B-sub"])
def test_project_lidar_tier1(SM, oracle_mod, config):
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=200_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config, seed=5 if config == "tiny" else None)
    r = lidar_run(SM, cfg, scene, write_all_records=True)
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    gv = np.isfinite(rec[:, 16])
    ov = proj["valid"] != 0
    amb = proj["ambiguous"] != 0
    assert np.array_equal(gv[~amb], ov[~amb]), np.nonzero(gv[~amb] != ov[~amb])[0][:10]
    both = gv & ov & ~amb
    # depth keys: bit-exact float32 (A19)
    assert np.array_equal(r.depth_key.cpu().numpy().view(np.uint32), proj["key"].view(np.uint32))
    db = np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both].astype(np.float64))
    print(f"box edge |gpu - oracle| max {db.max():.3e} p99.99 {np.percentile(db, 99.99):.3e}")
    assert db[:, :2].max() < LIDAR_EPS["a"] and db[:, 2:].max() < LIDAR_EPS["b"], db.max(0)
    Mref = proj["Mrows"][both]
    rel = np.abs(rec[both, 3:12] - Mref) / np.abs(Mref).max(1, keepdims=True)
    assert rel.max() < 2e-6
    assert np.abs(rec[both, 13:16] - proj["feat"][both]).max() < 2e-5


# ------------------------------------------------------------------ stages 3-4 (a2-a4): cull, pairs, sort
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("config", ["A", "tiny", "B-sub"])
def test_cull_bin_sort_tier1_bit_exact(SM, oracle_mod, config, mode):
    """Counts, tile rects, sorted (key, id) pairs and tile ranges bit-exact vs the oracle fed
    the GPU's boxes and keys; mode 1 = the paper's SAT culling, 2 = exact containment (A32)."""
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=300_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config, seed=9 if config == "tiny" else None)
    r = lidar_run(SM, cfg, scene, write_all_records=True, enable_culling=mode)
    t = O.Tiling(cfg)
    box = r.record.cpu().numpy()[:, 16:20].copy()
    valid = np.isfinite(box[:, 0]).astype(np.int32)
    count, rect = O.cull_lidar(valid, box, t, mode)
    assert np.array_equal(r.tile_count.cpu().numpy(), count)
    gr = r.tile_rect.cpu().numpy()
    nz = count > 0
    assert np.array_equal(gr[nz], rect[nz])
    keys, ids, ranges = O.bin_pairs(count, rect, r.depth_key.cpu().numpy(), t.n_tiles, t.n_theta)
    gk, gi, granges = sorted_lists(r)
    assert len(gk) == len(keys)
    assert np.array_equal(gk, keys) and np.array_equal(gi, ids) and np.array_equal(granges, ranges)


# ------------------------------------------------------------------ stage 5 (a5): compositing
@pytest.mark.parametrize("config", ["A", "tiny", "B-sub"])
def test_render_lidar_tier1(SM, oracle_mod, config):
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=300_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config, seed=11 if config == "tiny" else None)
    r = lidar_run(SM, cfg, scene)
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    rec = gpu_records(r)
    od = r.out["ray_od"].cpu().numpy()
    ref = O.composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, wrap=1, near=cfg.min_range,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    g, bd = O.decode_lidar(ref["feat"])
    ref["intensity"], ref["raydrop"] = g, bd
    ok = ref["flag"] == 0
    assert ok.mean() > 0.999, ok.mean()
    compare_lidar(r.out, ref, ok)
    assert (r.out["opacity"].cpu().numpy() > 0.5).mean() > 0.05  # the scan sees geometry


# ------------------------------------------------------------------ end to end (tier 2)
@pytest.mark.parametrize("config", ["A", "tiny"])
def test_lidar_end_to_end_tier2(SM, oracle_mod, config):
    O = oracle_mod
    cfg, scene = S.lidar_config(config), S.scene_for(config, seed=13 if config == "tiny" else None)
    r = lidar_run(SM, cfg, scene)
    t = O.Tiling(cfg)
    ref = O.render_lidar(scene, cfg, tiling=t, flag_eps=LIDAR_EPS)  # oracle rays (double), own projection
    ok = ref["flag"] == 0
    assert ok.mean() > 0.995, ok.mean()
    compare_lidar(r.out, ref, ok)
    brute = O.render_lidar(scene, cfg, tiling=t, mode="brute")  # O13: no tiling, no culling
    okb = ok
    compare_lidar(r.out, brute, okb)


def test_lidar_tiny_scenes_vs_bruteforce(SM, oracle_mod):
    O = oracle_mod
    worst = 0.0
    flagged = 0
    total = 0
    for seed in range(0, 100, 5):
        cfg, scene = S.lidar_config("tiny"), S.scene_for("tiny", seed=seed)
        r = lidar_run(SM, cfg, scene)
        ref = O.render_lidar(scene, cfg, mode="brute", flag_eps=LIDAR_EPS)
        ok = ref["flag"] == 0
        flagged += int((~ok).sum())
        total += ok.size
        e = compare_lidar(r.out, ref, ok)
        worst = max(worst, e["opacity"], e["intensity"])
    assert flagged / total < 0.005


# ------------------------------------------------------------------ invariance on the GPU alone
@pytest.mark.parametrize("config", ["B", "C"])
def test_gpu_invariance_tiling_and_culling(SM, config):
    scene = S.scene_for(config, n=200_000)
    outs = []
    for n_phi, M, cull in ((16, 32, 2), (16, 32, 1), (16, 32, 0), (8, 64, 1), (32, 16, 2), (4, 256, 1),
                           (1, 8, 2)):
        cfg = S.lidar_config(config)
        cfg.n_phi, cfg.max_rays_per_tile = n_phi, M
        r = lidar_run(SM, cfg, scene, enable_culling=cull)
        outs.append({k: v.cpu().numpy().copy() for k, v in r.out.items() if v is not None and k != "ray_od"})
    for o in outs[1:]:
        for k in outs[0]:
            assert np.array_equal(o[k], outs[0][k]), k  # tiling "does not affect quality"


@pytest.mark.parametrize("config", ["A", "tiny", "B-sub"])
def test_gpu_single_tile_bruteforce(SM, config):
    """GPU brute force ("does not affect quality"): one render tile holding every ray
    (N_phi = 1, M >= all rays, so N_theta = 1) and culling off, i.e. ONE list with every valid
    particle, tested by every ray -- bitwise equal to the default tiled, culled render."""
    name = "B" if config == "B-sub" else config
    scene = S.scene_for(name, n=50_000) if config == "B-sub" else S.scene_for(config, seed=5 if config == "tiny" else None)
    cfg = S.lidar_config(name)
    tiled = lidar_run(SM, cfg, scene)
    one = S.lidar_config(name)
    one.n_phi, one.max_rays_per_tile = 1, 1 << 30
    brute = lidar_run(SM, one, scene, enable_culling=0)
    assert brute.n_tiles == 1
    assert int(brute.n_pairs.item()) == int((brute.tile_count > 0).sum().item())  # every valid particle, once
    assert int(brute.n_pairs.item()) >= int((tiled.tile_count > 0).sum().item())
    for k, v in tiled.out.items():
        if v is not None:
            assert torch.equal(v, brute.out[k]), k


@pytest.mark.parametrize("per_ray_sh", [False, True])
def test_lidar_render_pipeline_shapes_identical(SM, per_ray_sh):
    """The LiDAR render's pipeline shapes (simuli_render_params.lidar_producers: 0 = hybrid,
    1..3 = producer / consumer, 4 = one warp per item) run the same responses and chain:
    outputs bit-identical (B subset, and tiles with more than 32 rays)."""
    for cfg_name, n_phi, M in (("B", 16, 32), ("A", 2, 128)):
        scene = S.scene_for(cfg_name, n=200_000) if cfg_name == "B" else S.scene_for(cfg_name)
        outs = []
        for prod in (0, 1, 2, 3, 4):
            cfg = S.lidar_config(cfg_name)
            cfg.n_phi, cfg.max_rays_per_tile = n_phi, M
            r = lidar_run(SM, cfg, scene, render_producers=prod, per_ray_sh=per_ray_sh)
            r.want_counters(True)
            r.render()
            torch.cuda.synchronize()
            outs.append({k: v.cpu().numpy().copy() for k, v in r.out.items() if v is not None})
        for o in outs[1:]:
            for k in outs[0]:
                assert np.array_equal(o[k], outs[0][k]), (cfg_name, k)


def test_scans_in_flight_deterministic(SM):
    """bench.py's regime: several renderers sharing one resident scene, scans enqueued on
    different streams concurrently -- every scan's outputs bit-identical to the same pose
    rendered alone, and the device-side pair-count check passes."""
    cfg = S.lidar_config("B")
    scene = SM.to_device_scene(S.scene_for("B", n=300_000))
    poses = S.batch_poses(512)[::97][:4]
    rs = [SM.LidarRenderer(cfg, scene) for _ in range(len(poses))]
    alone = SM.LidarRenderer(cfg, scene)
    ref = []
    for p0, p1 in poses:
        out = alone.scan(p0, p1, sync_capacity=True)
        torch.cuda.synchronize()
        ref.append({k: v.clone() for k, v in out.items() if v is not None})
    for r in rs:
        r.set_capacity(alone.capacity)
    streams = [torch.cuda.Stream() for _ in rs]
    for _ in range(2):  # twice, so each renderer's second scan overwrites its first
        for r, st, (p0, p1) in zip(rs, streams, poses):
            r.scan(p0, p1, stream=st)
    torch.cuda.synchronize()
    for r, want in zip(rs, ref):
        r.check_capacity()
        for k, v in want.items():
            assert torch.equal(r.out[k], v), k


@pytest.mark.parametrize("name", ["D-small", "pinhole-small"])
def test_camera_tile_size_invariance(SM, name):
    """Camera tiles of 8 and 16 px (A12 per-pixel box membership): outputs bit-identical."""
    scene = S.corridor_scene(7, 20000, x_range=(0.0, 40.0), kind="camera", ego=(1.5, 0.0, 1.6))
    outs = []
    for tp in (16, 8):
        cam = S.camera_config(name)
        cam.tile_px = tp
        c = camera_run(SM, cam, scene)
        outs.append({k: v.cpu().numpy().copy() for k, v in c.out.items() if v is not None and k != "ray_od"})
    for k in outs[0]:
        if k in ("n_visited",):  # list positions differ with the tiling; the rest must not
            continue
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_culling_reduces_pairs(SM):
    scene = S.scene_for("B", n=300_000)
    cfg = S.lidar_config("B")
    exact = lidar_run(SM, cfg, scene, enable_culling=2)
    on = lidar_run(SM, cfg, scene, enable_culling=1)
    off = lidar_run(SM, cfg, scene, enable_culling=0)
    assert on.n_pairs.item() < off.n_pairs.item()  # direction of tab:culling
    assert exact.n_pairs.item() < on.n_pairs.item()  # exact containment refines it (A32)


# ------------------------------------------------------------------ sort + edge cases
@pytest.mark.parametrize("skew", [False, True])
def test_bin_sort_synthetic_keys_large_tiles(SM, skew):
    """Stable sort of many pairs over 8160 tiles (13 tile bits) with many equal depth keys
    (ties by id), ragged last partition.  skew: ~60k pairs in one tile and ~3k in another."""
    dev = "cuda"
    rng = np.random.default_rng(17)
    n = 123_457
    n_tiles, ncols = 8160, 120
    count = rng.integers(0, 6, n).astype(np.int32)
    rect = np.zeros((n, 4), np.int32)
    rows = n_tiles // ncols
    r0 = rng.integers(0, rows, n)
    c0 = rng.integers(0, ncols, n)
    if skew:
        hot = rng.uniform(size=n)
        r0[hot < 0.5], c0[hot < 0.5] = 3, 7
        r0[(hot >= 0.5) & (hot < 0.525)], c0[(hot >= 0.5) & (hot < 0.525)] = 40, 119
    for i in range(n):
        h = int(rng.integers(1, 3))
        rect[i] = [r0[i], min(rows - 1, r0[i] + h - 1), c0[i], 1]
    count = ((rect[:, 1] - rect[:, 0] + 1) * rect[:, 3]).astype(np.int32)
    count[rng.uniform(size=n) < 0.2] = 0
    key = rng.choice(np.float32([0.5, 1.0, 2.0, 3.5]), n).astype(np.float32)  # many ties
    half = rng.uniform(size=n) < 0.5
    key[half] = rng.uniform(0.1, 200, int(half.sum())).astype(np.float32)
    t = {k: torch.from_numpy(v).to(dev) for k, v in (("count", count), ("rect", rect), ("key", key))}
    proj = SM.Projected(0, t["rect"].data_ptr(), t["key"].data_ptr(), t["count"].data_ptr())
    P = int(count.sum())
    cap = P + 17
    ws = torch.empty(SM.simuli_bin_sort_workspace_size(n, cap, n_tiles), dtype=torch.uint8, device=dev)
    keys = torch.empty(cap, dtype=torch.int64, device=dev)
    ids = torch.empty(cap, dtype=torch.int32, device=dev)
    ranges = torch.empty((n_tiles, 2), dtype=torch.int32, device=dev)
    npairs = torch.zeros(1, dtype=torch.int64, device=dev)
    torder = torch.empty(n_tiles, dtype=torch.int32, device=dev)
    SM.simuli_bin_sort(proj, n, n_tiles, ncols, ws, cap, keys, ids, ranges, npairs, tile_order=torder)
    torch.cuda.synchronize()
    assert npairs.item() == P
    # reference: enumerate pairs in particle order, stable sort by key
    g = np.repeat(np.arange(n), count)
    j = np.concatenate([np.arange(c) for c in count if c > 0])
    tile = (rect[g, 0] + j) * ncols + rect[g, 2]
    k64 = (tile.astype(np.uint64) << np.uint64(32)) | key.view(np.uint32)[g].astype(np.uint64)
    order = np.argsort(k64, kind="stable")
    assert np.array_equal(keys[:P].cpu().numpy().view(np.uint64), k64[order])
    assert np.array_equal(ids[:P].cpu().numpy(), g[order].astype(np.int32))
    rr = ranges.cpu().numpy()
    st = np.searchsorted(k64[order] >> np.uint64(32), np.arange(n_tiles), "left")
    en = np.searchsorted(k64[order] >> np.uint64(32), np.arange(n_tiles), "right")
    assert np.array_equal(rr[:, 0][en > st], st[en > st]) and np.array_equal(rr[:, 1], np.where(en > st, en, 0))
    od = torder.cpu().numpy()
    assert np.array_equal(np.sort(od), np.arange(n_tiles))  # a permutation, longest lists first
    lens = rr[od, 1] - rr[od, 0]
    assert np.all(np.diff(np.floor(np.log2(lens + 0.5))) <= 0)
    if skew:
        assert lens.max() > 16 * 2048


def test_bin_sort_capacity_protocol(SM):
    cfg, scene = S.lidar_config("A"), S.scene_for("A")
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), capacity=10)
    r.project()
    need = SM.simuli_bin_sort(r.projected, r.n, r.n_tiles, r.n_cols_total, r.workspace, -r.capacity, r.sorted_keys,
                              r.sorted_ids, r.tile_ranges, r.n_pairs)
    assert need is not None and need > 10
    SM.simuli_bin_sort(r.projected, r.n, r.n_tiles, r.n_cols_total, r.workspace, r.capacity, r.sorted_keys,
                       r.sorted_ids, r.tile_ranges, r.n_pairs)  # async: reports P, sorts a prefix
    torch.cuda.synchronize()
    assert r.n_pairs.item() == need
    r.scan(sync_capacity=True)  # grows and completes
    torch.cuda.synchronize()
    assert r.capacity >= need


def test_empty_and_degenerate_scenes(SM, oracle_mod):
    cfg = S.lidar_config("tiny")
    empty = {k: v[:0] for k, v in S.scene_for("tiny", seed=1).items()}
    r = SM.LidarRenderer(cfg, SM.to_device_scene(empty))
    out = r.scan(sync_capacity=True)
    torch.cuda.synchronize()
    assert (out["opacity"].cpu().numpy() == 0).all() and np.allclose(out["raydrop"].cpu().numpy(), 0.5)
    bad = S.scene_for("tiny", seed=2)
    n = bad["means"].shape[0]
    bad["quats"][: n // 3] = 0.0            # zero quaternion -> invalid
    bad["scales"][n // 3: n // 2, 0] = 0.0  # zero scale -> invalid
    bad["means"][n // 2: n // 2 + 3] = np.array([0, 0, 1.8], np.float32)  # at the sensor -> range < r_min
    r = lidar_run(SM, cfg, bad)
    ref = oracle_mod.render_lidar(bad, cfg, flag_eps=LIDAR_EPS)
    ok = ref["flag"] == 0
    compare_lidar(r.out, ref, ok)
    assert (r.tile_count.cpu().numpy()[: n // 2] == 0).all()


def test_many_rays_per_tile_chunks(SM, oracle_mod):
    """max_rays_in_tile > 32 (A9): warps over 32-ray chunks of one tile."""
    cfg = S.lidar_config("A")
    cfg.n_phi, cfg.max_rays_per_tile = 2, 128
    scene = S.scene_for("A")
    r = lidar_run(SM, cfg, scene)
    assert r.tiling_host["max_rays_in_tile"] > 32
    ref = oracle_mod.render_lidar(scene, cfg, flag_eps=LIDAR_EPS)
    compare_lidar(r.out, ref, ref["flag"] == 0)


# ------------------------------------------------------------------ full-size config B (sampled)
def _config_e_lidar():
    """Config E's parity scan: C-type sensor, the E scene (4M G_l), scan 17 of the E poses."""
    cfg = S.lidar_config("C")
    cfg.pose_start, cfg.pose_end = S.e_poses(64)[0][17]
    return cfg, S.scene_for("E-lidar")


@pytest.mark.parametrize("name", ["B", "C", "E"])
def test_lidar_full_size_sampled(SM, oracle_mod, name):
    """BASELINE configs[1] (B: Pandar64-like, 2M), configs[2] (C: Waymo-top-like, 4M) and one
    scan of configs[4] (E: C-type sensor in the E scene) at full size in the bench's launch
    configuration; the oracle checks the depth key of every particle and composites a sample
    of 64 tiles (tier 1 and tier 2)."""
    O = oracle_mod
    cfg, scene = _config_e_lidar() if name == "E" else (S.lidar_config(name), S.scene_for(name))
    r = lidar_run(SM, cfg, scene, write_all_records=False)
    keys = r.depth_key.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    assert np.array_equal(keys.view(np.uint32), proj["key"].view(np.uint32))
    t = O.Tiling(cfg)
    rng = np.random.default_rng(3)
    tiles = rng.choice(t.n_tiles, 64, replace=False)
    rays = np.concatenate([t.tile_rays[t.tile_ray_offsets[x]:t.tile_ray_offsets[x + 1]] for x in tiles])
    # tier 1 on the sample: GPU records / lists / rays
    _, ids, ranges = sorted_lists(r)
    rec = gpu_records(r)
    od = r.out["ray_od"].cpu().numpy()
    ref = O.composite(rec, ids, ranges, t.ray_tile[rays], t.ray_az[rays], t.ray_el[rays], od[rays], wrap=1,
                      near=cfg.min_range, flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref["intensity"], ref["raydrop"] = O.decode_lidar(ref["feat"])
    sub = {k: v[torch.from_numpy(rays).to(v.device)] for k, v in r.out.items() if v is not None}
    compare_lidar(sub, ref, ref["flag"] == 0)
    # tier 2 on the sample: oracle's own projection, lists and rays
    rec2 = O.records_from_projection(proj, scene)
    listed = ((proj["valid"] != 0) | (proj["ambiguous"] != 0)) & np.isfinite(proj["box"]).all(1)
    lbox = O.expand_box(proj["box"], LIDAR_EPS["a"], LIDAR_EPS["b"])
    amb = proj["ambiguous"] != 0
    lbox[amb] = O.expand_box(proj["box"][amb], *O.AMBIGUOUS_MARGIN)
    count, rect = O.cull_lidar(listed.astype(np.int32), lbox, t, False)
    _, ids2, ranges2 = O.bin_pairs(count, rect, proj["key"], t.n_tiles, t.n_theta)
    od2 = O.lidar_rays(t, cfg.pose_start, cfg.pose_end)[rays]
    gamb = np.where(proj["ambiguous"] != 0, np.where(proj["valid"] != 0, 1, 2), 0).astype(np.int32)
    ref2 = O.composite(rec2, ids2, ranges2, t.ray_tile[rays], t.ray_az[rays], t.ray_el[rays], od2, wrap=1,
                       near=cfg.min_range, gamb=gamb, flag_eps=LIDAR_EPS, pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref2["intensity"], ref2["raydrop"] = O.decode_lidar(ref2["feat"])
    ok = ref2["flag"] == 0
    assert ok.mean() > 1 - FLAG_BUDGET.get(name, FLAG_BUDGET["default"]), ok.mean()
    compare_lidar(sub, ref2, ok)


# ------------------------------------------------------------------ camera (a6)
def camera_run(SM, cam, scene, **kw):
    c = SM.CameraRenderer(cam, SM.to_device_scene(scene), **kw)
    c.want_ray_od(True)
    c.frame(sync_capacity=True)
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("name", ["D-small", "pinhole-small"])
def test_camera_tier1_and_tier2(SM, oracle_mod, name):
    O = oracle_mod
    cam = S.camera_config(name)
    scene = S.corridor_scene(21, 40000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6))
    c = camera_run(SM, cam, scene, write_all_records=True)
    rec = c.record.cpu().numpy()
    proj = O.project_camera(scene, cam)
    gv, ov, amb = np.isfinite(rec[:, 16]), proj["valid"] != 0, proj["ambiguous"] != 0
    assert np.array_equal(gv[~amb], ov[~amb])
    both = gv & ov
    db = np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both])
    print(f"camera box edge |gpu - oracle| max {db.max():.3e} px")
    assert db.max() < CAMERA_EPS["a"]
    count, rect = O.cull_camera(gv.astype(np.int32), rec[:, 16:20].copy(), cam)
    assert np.array_equal(c.tile_count.cpu().numpy(), count)
    Wt, Ht = O.camera_tiles(cam)
    keys, ids, ranges = O.bin_pairs(count, rect, c.depth_key.cpu().numpy(), Wt * Ht, Wt)
    gk, gi, gr = sorted_lists(c)
    assert np.array_equal(gk, keys) and np.array_equal(gi, ids) and np.array_equal(gr, ranges)
    rays = O.camera_rays(cam)
    gpu_od = c.out["ray_od"].cpu().numpy()
    assert np.abs(gpu_od - rays["od"])[rays["valid"] != 0].max() < 1e-9
    # tier 1: GPU records, lists, rays
    ref = O.composite(gpu_records(c), ids, ranges, rays["tile"], rays["u"], rays["v"], gpu_od, wrap=0,
                      near=cam.near, ray_valid=rays["valid"],
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4})
    ok = ref["flag"] == 0
    assert ok.mean() > 0.999
    rgb = c.out["rgb"].cpu().numpy()
    assert np.abs(rgb - ref["feat"])[ok].max() < TOL_FEAT
    assert np.abs(c.out["opacity"].cpu().numpy() - ref["opacity"])[ok].max() < TOL_FEAT
    # tier 2: oracle from scratch
    ref2 = O.render_camera(scene, cam, flag_eps=CAMERA_EPS)
    ok2 = ref2["flag"] == 0
    assert ok2.mean() > 0.995, ok2.mean()
    assert np.abs(rgb - ref2["feat"])[ok2].max() < TOL_FEAT
    dm = ok2 & (ref2["opacity"] >= 0.5)
    assert np.abs(c.out["depth"].cpu().numpy() - ref2["depth"])[dm].max() < TOL_DEPTH
    assert (c.out["opacity"].cpu().numpy() > 0.1).mean() > 0.05


@pytest.mark.parametrize("name", ["D", "E"])
def test_camera_config_d_full_size_sampled(SM, oracle_mod, name):
    """BASELINE configs[3]: KB fisheye rolling-shutter 1920x1080, 2M particles, at full size
    (and one frame of configs[4]: a D-type frame of the E scene, 4M G_c, frame 17).  Every
    particle's box / validity / depth key is checked; 48 random 16x16 tiles are composited by
    the oracle, tier 1 (GPU records, lists, rays) and tier 2 (oracle's own)."""
    O = oracle_mod
    cam = S.camera_config("D")
    if name == "E":
        cam.pose_start, cam.pose_end = S.e_poses(64)[1][17]
        scene = S.scene_for("E-camera")
    else:
        scene = S.scene_for("D")
    c = camera_run(SM, cam, scene, write_all_records=True)
    rec = c.record.cpu().numpy()
    proj = O.project_camera(scene, cam)
    gv, ov, amb = np.isfinite(rec[:, 16]), proj["valid"] != 0, proj["ambiguous"] != 0
    assert np.array_equal(gv[~amb], ov[~amb])
    assert np.array_equal(c.depth_key.cpu().numpy().view(np.uint32), proj["key"].view(np.uint32))
    both = gv & ov & ~amb
    assert np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both]).max() < CAMERA_EPS["a"]
    Wt, Ht = O.camera_tiles(cam)
    rays = O.camera_rays(cam)
    rng = np.random.default_rng(4)
    tiles = rng.choice(Wt * Ht, 48, replace=False)
    sel = np.nonzero(np.isin(rays["tile"], tiles))[0]
    gpu_od = c.out["ray_od"].cpu().numpy()
    _, gi, gr = sorted_lists(c)
    sub = lambda d: {k: (v[sel] if isinstance(v, np.ndarray) and v.shape[:1] == (cam.width * cam.height,) else v)
                     for k, v in d.items()}
    rs = sub(rays)
    ref = O.composite(gpu_records(c), gi, gr, rs["tile"], rs["u"], rs["v"], gpu_od[sel], wrap=0, near=cam.near,
                      ray_valid=rs["valid"], flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4})
    ok = ref["flag"] == 0
    assert ok.mean() > 0.999
    rgb = c.out["rgb"].cpu().numpy()[sel]
    assert np.abs(rgb - ref["feat"])[ok].max() < TOL_FEAT
    # tier 2: the oracle's own projection, lists and rays on the sample
    rec2 = O.records_from_projection(proj, scene)
    listed = ((proj["valid"] != 0) | (proj["ambiguous"] != 0)) & np.isfinite(proj["box"]).all(1)
    lbox = O.expand_box(proj["box"], CAMERA_EPS["a"], CAMERA_EPS["b"])
    lbox[amb] = O.expand_box(proj["box"][amb], CAMERA_EPS["amb_a"], CAMERA_EPS["amb_b"])
    count, rect = O.cull_camera(listed.astype(np.int32), lbox, cam)
    _, ids2, ranges2 = O.bin_pairs(count, rect, proj["key"], Wt * Ht, Wt)
    gamb = np.where(amb, np.where(proj["valid"] != 0, 1, 2), 0).astype(np.int32)
    ref2 = O.composite(rec2, ids2, ranges2, rs["tile"], rs["u"], rs["v"], rs["od"], wrap=0, near=cam.near,
                       ray_valid=rs["valid"], gamb=gamb, flag_eps=CAMERA_EPS)
    ok2 = ref2["flag"] == 0
    assert ok2.mean() > 1 - FLAG_BUDGET["default"], ok2.mean()
    assert np.abs(rgb - ref2["feat"])[ok2].max() < TOL_FEAT
    dm = ok2 & (ref2["opacity"] >= 0.5)
    assert np.abs(c.out["depth"].cpu().numpy()[sel] - ref2["depth"])[dm].max(initial=0) < TOL_DEPTH
    assert (c.out["opacity"].cpu().numpy() > 0.1).mean() > 0.05


# ------------------------------------------------------------------ beam divergence (NEXT-2)
@pytest.mark.parametrize("config", ["A", "B-sub"])
def test_beam_divergence_parity(SM, oracle_mod, config):
    """App. C filter (theta_div = 1.5e-3 rad, SPEC S:287's value; A24/A27) on the GPU path:
    projection (boxes, canonical transform from chol(Sigma_hat)^-1), then compositing tier 1
    (GPU records / lists / rays) and tier 2 (oracle from scratch, A23 flags)."""
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=200_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config)
    cfg.beam_divergence = 1.5e-3
    r = lidar_run(SM, cfg, scene, write_all_records=True)
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    gv, ov, amb = np.isfinite(rec[:, 16]), proj["valid"] != 0, proj["ambiguous"] != 0
    assert np.array_equal(gv[~amb], ov[~amb])
    both = gv & ov & ~amb
    db = np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both])
    assert db[:, :2].max() < LIDAR_EPS["a"] and db[:, 2:].max() < LIDAR_EPS["b"], db.max(0)
    Mref = proj["Mrows"][both]
    rel = np.abs(rec[both, 3:12] - Mref) / np.abs(Mref).max(1, keepdims=True)
    assert rel.max() < 2e-5, rel.max()
    # the filter changed the particles (not a silent no-op)
    cfg0 = S.lidar_config("B" if config == "B-sub" else config)
    assert not np.array_equal(O.project_lidar(scene, cfg0)["Mrows"][both], Mref)
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    od = r.out["ray_od"].cpu().numpy()
    ref = O.composite(gpu_records(r), ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, wrap=1, near=cfg.min_range,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref["intensity"], ref["raydrop"] = O.decode_lidar(ref["feat"])
    ok = ref["flag"] == 0
    assert ok.mean() > 0.999
    compare_lidar(r.out, ref, ok)
    if config == "A":
        ref2 = O.render_lidar(scene, cfg, tiling=t, flag_eps=LIDAR_EPS)
        ok2 = ref2["flag"] == 0
        assert ok2.mean() > 1 - FLAG_BUDGET["default"], ok2.mean()
        compare_lidar(r.out, ref2, ok2)


# ------------------------------------------------------------------ sensor-model variants
@pytest.mark.parametrize("variant", ["cw_spin", "K2", "K0", "az_start", "static_pose", "rotating_fast", "tilted"])
def test_lidar_sensor_variants(SM, oracle_mod, variant):
    """Paths of the sensor model the BASELINE configs do not exercise: clockwise spin,
    K = 2 and K = 0 firing-time iterations (A3), a non-default phi_start, a static pose, and
    a fast-rotating sweep (0.6 rad of yaw: the general rotation branch instead of the
    small-angle series), and a sweep rotating about a tilted axis (the general Rodrigues form
    of the sigma-point offsets instead of the planar yaw-only one).  Tier 1 projection +
    compositing and tier 2 end to end on config A
    geometry (32 x 512 rays, 1k particles) moved through a 1.5 m / yawing sweep."""
    O = oracle_mod
    cfg, scene = S.lidar_config("A"), S.scene_for("A")
    cfg.pose_start = S.pose(S.yaw_quat(0.1), [0.0, 0.0, 1.8])
    cfg.pose_end = S.pose(S.yaw_quat(0.13), [1.5, 0.3, 1.8])
    if variant == "cw_spin":
        cfg.spin_direction = -1
    elif variant == "K2":
        cfg.rs_iterations = 2
    elif variant == "K0":
        cfg.rs_iterations = 0
    elif variant == "az_start":
        cfg.azimuth_start = float(np.float32(0.7))
    elif variant == "static_pose":
        cfg.pose_end = cfg.pose_start
    elif variant == "rotating_fast":
        cfg.pose_end = S.pose(S.yaw_quat(0.7), [1.5, 0.3, 1.8])
    elif variant == "tilted":  # 0.05 rad about (0.1, 0.2, 1) after the start yaw
        ax = np.array([0.1, 0.2, 1.0]) / np.linalg.norm([0.1, 0.2, 1.0])
        qt = np.concatenate([[np.cos(0.025)], np.sin(0.025) * ax])
        q0 = np.asarray(S.yaw_quat(0.1), np.float64)
        w1, x1, y1, z1 = q0
        w2, x2, y2, z2 = qt
        q1 = [w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
              w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2]
        cfg.pose_end = S.pose(q1, [1.5, 0.3, 1.8])
    r = lidar_run(SM, cfg, scene, write_all_records=True)
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    gv, ov, amb = np.isfinite(rec[:, 16]), proj["valid"] != 0, proj["ambiguous"] != 0
    assert np.array_equal(gv[~amb], ov[~amb])
    both = gv & ov & ~amb
    db = np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both])
    assert db[:, :2].max() < LIDAR_EPS["a"] and db[:, 2:].max() < LIDAR_EPS["b"], db.max(0)
    assert np.array_equal(r.depth_key.cpu().numpy().view(np.uint32), proj["key"].view(np.uint32))
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    od = r.out["ray_od"].cpu().numpy()
    ref = O.composite(gpu_records(r), ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, wrap=1, near=cfg.min_range,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref["intensity"], ref["raydrop"] = O.decode_lidar(ref["feat"])
    ok = ref["flag"] == 0
    assert ok.mean() > 0.999
    compare_lidar(r.out, ref, ok)
    ref2 = O.render_lidar(scene, cfg, tiling=t, flag_eps=LIDAR_EPS)
    ok2 = ref2["flag"] == 0
    assert ok2.mean() > 1 - FLAG_BUDGET["default"], ok2.mean()
    compare_lidar(r.out, ref2, ok2)


@pytest.mark.parametrize("variant", ["global_shutter", "K2", "kb_static", "radtan_rolling", "tile8"])
def test_camera_variants(SM, oracle_mod, variant):
    """Camera paths beyond D: global shutter, K = 2 row fixed point, a static KB camera,
    pinhole-radtan with rolling shutter, 8x8-pixel tiles; tier 2 (oracle from scratch) on
    320 x 180 frames."""
    O = oracle_mod
    cam = S.camera_config("pinhole-small" if variant == "radtan_rolling" else "D-small")
    if variant == "global_shutter":
        cam.rolling_shutter = 0
    elif variant == "K2":
        cam.rs_iterations = 2
    elif variant == "kb_static":
        cam.pose_end = cam.pose_start
    elif variant == "tile8":
        cam.tile_px = 8
    scene = S.corridor_scene(23, 30000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6))
    c = camera_run(SM, cam, scene)
    ref = O.render_camera(scene, cam, flag_eps=CAMERA_EPS)
    ok = ref["flag"] == 0
    assert ok.mean() > 0.995, ok.mean()
    rgb = c.out["rgb"].cpu().numpy()
    assert np.abs(rgb - ref["feat"])[ok].max() < TOL_FEAT
    assert np.abs(c.out["opacity"].cpu().numpy() - ref["opacity"])[ok].max() < TOL_FEAT
    dm = ok & (ref["opacity"] >= 0.5)
    assert np.abs(c.out["depth"].cpu().numpy() - ref["depth"])[dm].max(initial=0) < TOL_DEPTH


@pytest.mark.parametrize("degree", [0, 1, 2])
def test_lower_sh_degrees(SM, oracle_mod, degree):
    """SH degrees below 3 (the generic feature path): features per particle and the
    composited outputs, tier 1, on config A with the coefficients truncated to (d+1)^2."""
    O = oracle_mod
    cfg, scene = S.lidar_config("A"), dict(S.scene_for("A"))
    scene["sh"] = np.ascontiguousarray(scene["sh"][:, : (degree + 1) ** 2, :])
    r = lidar_run(SM, cfg, scene, write_all_records=True)
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    both = np.isfinite(rec[:, 16]) & (proj["valid"] != 0) & (proj["ambiguous"] == 0)
    assert np.abs(rec[both, 13:16] - proj["feat"][both]).max() < 2e-5
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    ref = O.composite(gpu_records(r), ids, ranges, t.ray_tile, t.ray_az, t.ray_el, r.out["ray_od"].cpu().numpy(),
                      wrap=1, near=cfg.min_range, flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4,
                                                            "tau": 1e-4}, pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref["intensity"], ref["raydrop"] = O.decode_lidar(ref["feat"])
    compare_lidar(r.out, ref, ref["flag"] == 0)


@pytest.mark.parametrize("name", ["D-small", "pinhole-small"])
def test_compose_camera_parity(SM, oracle_mod, name):
    """Eq. 2 (P: camera model, A28): GPU simuli_compose_camera vs the oracle's compose on the
    same c_f / omega (the GPU frame's), with a random environment map and a random
    near-identity bilateral grid; also env only, grid only and neither."""
    O = oracle_mod
    cam = S.camera_config(name)
    scene = S.corridor_scene(23, 20000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6))
    c = camera_run(SM, cam, scene)
    rng = np.random.default_rng(77)
    env = rng.uniform(0, 1, (32, 64, 3)).astype(np.float32)
    grid = np.zeros((8, 9, 16, 12), np.float32)
    grid[..., 0] = grid[..., 5] = grid[..., 10] = 1.0
    grid += rng.normal(scale=0.05, size=grid.shape).astype(np.float32)
    rays = O.camera_rays(cam)
    cf = c.out["rgb"].cpu().numpy().astype(np.float64)
    om = c.out["opacity"].cpu().numpy().astype(np.float64)
    assert (om > 0.1).mean() > 0.02 and (om < 0.9).mean() > 0.02
    valid = rays["valid"] != 0
    for e, g in ((env, grid), (env, None), (None, grid), (None, None)):
        got = c.compose(None if e is None else torch.from_numpy(e).cuda(),
                        None if g is None else torch.from_numpy(g).cuda()).cpu().numpy()
        ref = O.compose_camera(cam, rays["od"], cf, om, e, g)
        err = np.abs(got - ref)[valid].max()
        print(f"{name} env={e is not None} grid={g is not None}: max |gpu - oracle| {err:.2e}")
        assert err < 2e-5
        if e is None:
            assert np.abs(got - ref).max() < 2e-5  # invalid pixels: no background term at all


# ------------------------------------------------------------------ scene graph (A29)
def test_actor_scene_lidar_parity(SM, oracle_mod):
    """Dynamic objects in local frames + poses at t: the GPU projection maps them to world
    (A29) -- depth keys bit-exact against the oracle's world means (O0), boxes / M / f
    within the tier-1 tolerances, lists bit-exact, and the whole scan within tier 2."""
    O = oracle_mod
    cfg = S.lidar_config("B")
    scene = S.with_actors(S.corridor_scene(41, 60_000, x_range=(-60.0, 60.0)), 42, n_actors=12, per_actor=2000,
                          x_range=(-40.0, 40.0))
    scene["actor_id"][:5] = [12, -3, 99, 12, 1000]  # out of range -> invalid
    r = lidar_run(SM, cfg, scene, write_all_records=True)
    rec = r.record.cpu().numpy()
    proj = O.project_lidar(scene, cfg)
    gv, ov, amb = np.isfinite(rec[:, 16]), proj["valid"] != 0, proj["ambiguous"] != 0
    assert not gv[:5].any() and not ov[:5].any()
    assert np.array_equal(gv[~amb], ov[~amb])
    assert np.array_equal(r.depth_key.cpu().numpy().view(np.uint32), proj["key"].view(np.uint32))
    both = gv & ov & ~amb
    world = O.actors_to_world(scene)
    assert np.array_equal(rec[both, 0:3], world["means"][both])  # record mu = the world mean
    db = np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both].astype(np.float64))
    assert db[:, :2].max() < LIDAR_EPS["a"] and db[:, 2:].max() < LIDAR_EPS["b"], db.max(0)
    Mref = proj["Mrows"][both]
    assert (np.abs(rec[both, 3:12] - Mref) / np.abs(Mref).max(1, keepdims=True)).max() < 2e-6
    moving = both & (scene["actor_id"] >= 0)
    assert moving.sum() > 1000
    t = O.Tiling(cfg)
    ref = O.render_lidar(scene, cfg, tiling=t, flag_eps=LIDAR_EPS)
    ok = ref["flag"] == 0
    assert ok.mean() > 1 - FLAG_BUDGET["default"], ok.mean()
    compare_lidar(r.out, ref, ok)


def test_actor_scene_camera_parity(SM, oracle_mod):
    O = oracle_mod
    cam = S.camera_config("D-small")
    scene = S.with_actors(S.corridor_scene(43, 30_000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6)), 44,
                          n_actors=6, per_actor=1500, kind="camera")
    c = camera_run(SM, cam, scene, write_all_records=True)
    rec = c.record.cpu().numpy()
    proj = O.project_camera(scene, cam)
    gv, ov, amb = np.isfinite(rec[:, 16]), proj["valid"] != 0, proj["ambiguous"] != 0
    assert np.array_equal(gv[~amb], ov[~amb])
    both = gv & ov
    assert np.abs(rec[both, 16:20].astype(np.float64) - proj["box"][both]).max() < CAMERA_EPS["a"]
    ref2 = O.render_camera(scene, cam, flag_eps=CAMERA_EPS)
    ok2 = ref2["flag"] == 0
    assert ok2.mean() > 0.995, ok2.mean()
    assert np.abs(c.out["rgb"].cpu().numpy() - ref2["feat"])[ok2].max() < TOL_FEAT
    seen = np.unique(scene["actor_id"][both & (scene["actor_id"] >= 0)])
    assert len(seen) >= 3


# ------------------------------------------------------------------ per-ray SH (Eq. 1 literally, A30)
@pytest.mark.parametrize("config", ["A", "B-sub"])
def test_per_ray_sh_lidar_parity(SM, oracle_mod, config):
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=200_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config)
    r = lidar_run(SM, cfg, scene, per_ray_sh=True)
    ref = O.render_lidar(scene, cfg, flag_eps=LIDAR_EPS, per_ray_sh=True)
    ok = ref["flag"] == 0
    assert ok.mean() > 1 - FLAG_BUDGET["default"], ok.mean()
    e = compare_lidar(r.out, ref, ok)
    print(config, e)
    base = lidar_run(SM, cfg, scene)  # per-particle features: same weights, other zeta
    assert torch.equal(base.out["opacity"], r.out["opacity"])
    assert (base.out["zeta"] - r.out["zeta"]).abs().max().item() > 1e-4


def test_per_ray_sh_camera_parity(SM, oracle_mod):
    O = oracle_mod
    cam = S.camera_config("D-small")
    scene = S.corridor_scene(21, 40000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6))
    c = camera_run(SM, cam, scene, per_ray_sh=True)
    ref2 = O.render_camera(scene, cam, flag_eps=CAMERA_EPS, per_ray_sh=True)
    ok2 = ref2["flag"] == 0
    assert ok2.mean() > 0.995, ok2.mean()
    err = np.abs(c.out["rgb"].cpu().numpy() - ref2["feat"])[ok2].max()
    print("camera per-ray SH max |gpu - oracle|", err)
    assert err < TOL_FEAT


# ------------------------------------------------------------------ backward (O15, O16; A31)
def _compare_grads(gpu, ref, what):
    for k in ("means", "quats", "scales", "opacity", "sh"):
        a = gpu[k].cpu().numpy().astype(np.float64).reshape(ref[k].shape)
        b = ref[k]
        scale = np.abs(b).max()
        assert scale > 0, (what, k)
        err = np.abs(a - b)
        print(f"{what} d{k}: max |gpu - oracle| / max |oracle| = {err.max() / scale:.2e}")
        assert err.max() <= 1e-3 * scale, (what, k, err.max(), scale)
        big = np.abs(b) > 1e-2 * scale
        assert (err[big] <= 1e-3 * np.abs(b[big]) + 1e-5 * scale).mean() > 0.999, (what, k)


def _upstream(R, seed, lidar, mask):
    rng = np.random.default_rng(seed)
    m = mask.astype(np.float64)
    g = {"opacity": rng.normal(size=R) * m, "depth_accum": 0.05 * rng.normal(size=R) * m,
         "depth": 0.05 * rng.normal(size=R) * m}
    if lidar:
        g.update({"zeta": rng.normal(size=(R, 3)) * m[:, None], "intensity": rng.normal(size=R) * m,
                  "raydrop": rng.normal(size=R) * m})
    else:
        g["rgb"] = rng.normal(size=(R, 3)) * m[:, None]
    return g


def _dev(g):
    return {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda() for k, v in g.items()}


@pytest.mark.parametrize("config", ["A", "B-sub"])
def test_backward_lidar_parity(SM, oracle_mod, config):
    """GPU backward vs the oracle's O15/O16 on the GPU's own records, lists and rays (tier 1);
    rays the tier-1 forward flags near a threshold get zero upstream gradient on both sides.
    Config A also tier 2 (the oracle's own forward)."""
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=200_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config)
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
    r.requires_grad(True)
    r.want_ray_od(True)
    r.scan(sync_capacity=True)
    torch.cuda.synchronize()
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    rec = gpu_records(r)
    od = r.out["ray_od"].cpu().numpy()
    fwd = O.composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, wrap=1, near=cfg.min_range,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ok = fwd["flag"] == 0
    R = od.shape[0]
    g = _upstream(R, 5, True, ok)
    got = r.backward(_dev(g))
    got_p1 = r.backward(_dev(g), use_forward_totals=False)  # the backward's own totals pass
    torch.cuda.synchronize()
    for k in got:
        assert torch.allclose(got[k], got_p1[k], rtol=1e-4, atol=1e-6 * got[k].abs().max().item()), k
    gz, go, gd = O.fold_upstream(fwd, g, lidar=True)
    d = O.backward_composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, gz, go, gd, wrap=1,
                             near=cfg.min_range, pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref = O.backward_params(scene, {"viewdir": r.view_dir.cpu().numpy().astype(np.float64)}, d)
    _compare_grads(got, ref, f"{config} tier 1")
    if config == "A":
        ref2f = O.render_lidar(scene, cfg, tiling=t, flag_eps=LIDAR_EPS)
        ok2 = (ref2f["flag"] == 0) & ok
        g2 = _upstream(R, 6, True, ok2)
        got2 = r.backward(_dev(g2))
        torch.cuda.synchronize()
        ref2 = O.backward_lidar(scene, cfg, g2, tiling=t)
        _compare_grads(got2, ref2, f"{config} tier 2")


@pytest.mark.parametrize("variant", ["D-small", "tile8_deg1", "pinhole_deg2"])
def test_backward_camera_parity(SM, oracle_mod, variant):
    O = oracle_mod
    cam = S.camera_config("pinhole-small" if variant == "pinhole_deg2" else "D-small")
    scene = S.corridor_scene(21, 40000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6))
    if variant == "tile8_deg1":
        cam.tile_px = 8
        scene["sh"] = np.ascontiguousarray(scene["sh"][:, :4])
    elif variant == "pinhole_deg2":
        scene["sh"] = np.ascontiguousarray(scene["sh"][:, :9])
    c = SM.CameraRenderer(cam, SM.to_device_scene(scene))
    c.requires_grad(True)
    c.want_ray_od(True)
    c.frame(sync_capacity=True)
    torch.cuda.synchronize()
    _, ids, ranges = sorted_lists(c)
    rays = O.camera_rays(cam)
    rec = gpu_records(c)
    od = c.out["ray_od"].cpu().numpy()
    fwd = O.composite(rec, ids, ranges, rays["tile"], rays["u"], rays["v"], od, wrap=0, near=cam.near,
                      ray_valid=rays["valid"], flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4,
                                                         "tau": 1e-4})
    ok = fwd["flag"] == 0
    g = _upstream(od.shape[0], 7, False, ok)
    got = c.backward(_dev(g))
    torch.cuda.synchronize()
    gz, go, gd = O.fold_upstream(fwd, g, lidar=False)
    d = O.backward_composite(rec, ids, ranges, rays["tile"], rays["u"], rays["v"], od, gz, go, gd, wrap=0,
                             near=cam.near, ray_valid=rays["valid"])
    ref = O.backward_params(scene, {"viewdir": c.view_dir.cpu().numpy().astype(np.float64)}, d)
    _compare_grads(got, ref, f"{variant} tier 1")


def test_backward_empty(SM):
    """n = 0 is a no-op."""
    cfg = S.lidar_config("A")
    sc = {k: v[:0] for k, v in S.scene_for("A").items()}
    r = SM.LidarRenderer(cfg, SM.to_device_scene(sc))
    r.requires_grad(True)
    r.scan(sync_capacity=True)
    out = r.backward({"opacity": torch.ones(r.n_rays, device="cuda")})
    torch.cuda.synchronize()
    assert out["means"].numel() == 0


@pytest.mark.parametrize("config", ["A", "B-sub"])
def test_backward_beam_divergence_parity(SM, oracle_mod, config):
    """Backward with the App. C filter (A27, A31): M = chol(Sigma_hat)^-1 through the
    Cholesky factor and the view vector, tier 1 against O15/O16."""
    O = oracle_mod
    if config == "B-sub":
        cfg, scene = S.lidar_config("B"), S.scene_for("B", n=200_000)
    else:
        cfg, scene = S.lidar_config(config), S.scene_for(config)
    cfg.beam_divergence = 1.5e-3
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
    r.requires_grad(True)
    r.want_ray_od(True)
    r.scan(sync_capacity=True)
    torch.cuda.synchronize()
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    rec = gpu_records(r)
    od = r.out["ray_od"].cpu().numpy()
    fwd = O.composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, wrap=1, near=cfg.min_range,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    g = _upstream(od.shape[0], 13, True, fwd["flag"] == 0)
    got = r.backward(_dev(g))
    torch.cuda.synchronize()
    gz, go, gd = O.fold_upstream(fwd, g, lidar=True)
    d = O.backward_composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, gz, go, gd, wrap=1,
                             near=cfg.min_range, pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref = O.backward_params(scene, {"viewdir": r.view_dir.cpu().numpy().astype(np.float64)}, d,
                            beam_div=cfg.beam_divergence)
    _compare_grads(got, ref, f"divergence {config} tier 1")


@pytest.mark.parametrize("sensor", ["lidar", "camera"])
def test_backward_per_ray_sh_parity(SM, oracle_mod, sensor):
    """Per-ray SH backward (A30, A31): SH gradients summed over rays with the ray's basis,
    tier 1 against O15 with the same records, lists and rays."""
    O = oracle_mod
    if sensor == "lidar":
        cfg, scene = S.lidar_config("A"), S.scene_for("A")
        f = SM.LidarRenderer(cfg, SM.to_device_scene(scene), per_ray_sh=True)
        f.requires_grad(True)
        f.want_ray_od(True)
        f.scan(sync_capacity=True)
        t = O.Tiling(cfg)
        ray_tile, ra, rb, rv, kw = t.ray_tile, t.ray_az, t.ray_el, None, dict(wrap=1, near=cfg.min_range,
                                                                               pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    else:
        cam = S.camera_config("D-small")
        scene = S.corridor_scene(21, 40000, x_range=(0.0, 50.0), kind="camera", ego=(1.5, 0.0, 1.6))
        f = SM.CameraRenderer(cam, SM.to_device_scene(scene), per_ray_sh=True)
        f.requires_grad(True)
        f.want_ray_od(True)
        f.frame(sync_capacity=True)
        rays = O.camera_rays(cam)
        ray_tile, ra, rb, rv, kw = rays["tile"], rays["u"], rays["v"], rays["valid"], dict(wrap=0, near=cam.near)
    torch.cuda.synchronize()
    _, ids, ranges = sorted_lists(f)
    rec = gpu_records(f)
    rec["sh"] = scene["sh"]
    od = f.out["ray_od"].cpu().numpy()
    fwd = O.composite(rec, ids, ranges, ray_tile, ra, rb, od, ray_valid=rv,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4}, **kw)
    g = _upstream(od.shape[0], 11, sensor == "lidar", fwd["flag"] == 0)
    got = f.backward(_dev(g))
    torch.cuda.synchronize()
    gz, go, gd = O.fold_upstream(fwd, g, lidar=sensor == "lidar")
    d = O.backward_composite(rec, ids, ranges, ray_tile, ra, rb, od, gz, go, gd, ray_valid=rv, **kw)
    ref = O.backward_params(scene, {"viewdir": f.view_dir.cpu().numpy().astype(np.float64)}, d)
    _compare_grads(got, ref, f"per-ray SH {sensor} tier 1")


def test_backward_segmented_walk(SM, oracle_mod):
    """Lists longer than one 1024-entry segment (config A sensor, 150k particles): the
    segmented walk (stats pass + gradient pass from the earlier segments' transmittance and
    sums) against the unsegmented walk and against O15/O16 (tier 1)."""
    O = oracle_mod
    cfg, scene = S.lidar_config("A"), S.scene_for("A", n=150_000)
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene))
    r.requires_grad(True)
    r.want_ray_od(True)
    r.scan(sync_capacity=True)
    torch.cuda.synchronize()
    lens = np.diff(r.tile_ranges.cpu().numpy(), axis=1)
    assert lens.max() > 1024, lens.max()  # at least two segments
    t = O.Tiling(cfg)
    _, ids, ranges = sorted_lists(r)
    rec = gpu_records(r)
    od = r.out["ray_od"].cpu().numpy()
    fwd = O.composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, wrap=1, near=cfg.min_range,
                      flag_eps={"a": 0.0, "b": 0.0, "alpha": 2e-7, "T_rel": 1e-4, "tau": 1e-4},
                      pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    g = _upstream(od.shape[0], 12, True, fwd["flag"] == 0)
    seg = r.backward(_dev(g))
    whole = r.backward(_dev(g), use_forward_totals=False)
    torch.cuda.synchronize()
    for k in seg:
        a, b = seg[k].cpu().numpy(), whole[k].cpu().numpy()
        assert np.abs(a - b).max() <= 1e-4 * np.abs(b).max(), k
    gz, go, gd = O.fold_upstream(fwd, g, lidar=True)
    d = O.backward_composite(rec, ids, ranges, t.ray_tile, t.ray_az, t.ray_el, od, gz, go, gd, wrap=1,
                             near=cfg.min_range, pi_f=t.pi_f, two_pi_f=t.two_pi_f)
    ref = O.backward_params(scene, {"viewdir": r.view_dir.cpu().numpy().astype(np.float64)}, d)
    _compare_grads(seg, ref, "segmented tier 1")


def _scaled(scene, f):
    out = dict(scene)
    out["means"] = scene["means"] * np.float32(f)
    out["scales"] = scene["scales"] * np.float32(f)
    return out


@pytest.mark.parametrize("kind", ["lidar-B", "camera-D"])
def test_gpu_full_size_scale_covariance(SM, kind):
    """Full-size property check of the CUDA path (configs B and D, the bench's launch
    configuration): the render is a function of lengths only through dimensionless ratios
    (Eq. 3 sees directions, the canonical response and the depth order are homogeneous), and
    scaling every length by 2 is exact in binary floating point -- so the 2x scene seen from
    the 2x sensor track returns depth x 2 and every other output bit for bit (the oracle is
    pinned to the same property, test_oracle_pins.test_whole_*_scale_covariance)."""
    import copy
    if kind == "lidar-B":
        cfg = S.lidar_config("B")
        scene = S.scene_for("B")
        scene["means"] = (scene["means"] - np.float32([0.0, 0.0, 1.8])).astype(np.float32)
        cfg.pose_start, cfg.pose_end = S.pose([1, 0, 0, 0], [0, 0, 0]), S.pose(S.yaw_quat(0.03), [1.0, 0, 0])
        cfg2 = copy.deepcopy(cfg)
        cfg2.min_range = cfg.min_range * 2
        cfg2.pose_end = S.pose(S.yaw_quat(0.03), [2.0, 0, 0])
        a, b = lidar_run(SM, cfg, scene), lidar_run(SM, cfg2, _scaled(scene, 2))
        assert (a.out["opacity"] > 0.5).float().mean().item() > 0.2
    else:
        cfg = S.camera_config("D")
        scene = S.scene_for("D")
        scene["means"] = (scene["means"] - np.float32([1.5, 0.0, 1.6])).astype(np.float32)
        cfg.pose_start = S.pose(S.CAM_FORWARD_Q, [0, 0, 0])
        cfg.pose_end = S.pose(S.yaw_quat(0.009, S.CAM_FORWARD_Q), [0.3, 0, 0])
        cfg2 = copy.deepcopy(cfg)
        cfg2.near = cfg.near * 2
        cfg2.pose_end = S.pose(S.yaw_quat(0.009, S.CAM_FORWARD_Q), [0.6, 0, 0])
        a, b = camera_run(SM, cfg, scene), camera_run(SM, cfg2, _scaled(scene, 2))
        assert (a.out["opacity"] > 0.2).float().mean().item() > 0.1
    assert int(a.n_pairs.item()) == int(b.n_pairs.item())
    for k, v in a.out.items():
        if v is None:
            continue
        w = b.out[k]
        if k in ("depth", "depth_accum"):
            assert torch.equal(w, 2 * v), k
        elif k == "ray_od":
            assert torch.equal(w[..., :3], 2 * v[..., :3]) and torch.equal(w[..., 3:], v[..., 3:]), k
        else:
            assert torch.equal(w, v), k
