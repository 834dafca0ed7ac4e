"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
libsimuli kernel family on config A and a 200k-particle config-B subset -- LiDAR forward
(SAT and exact culling), beam divergence, per-ray SH, scene graph, LiDAR backward; camera
D-small forward, Eq. 2 compose and backward.  No oracle, no checks of values: the sanitizer
reports memory / race / sync / init errors.  Usage: python scripts/sanitize_run.py [--quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_12901_b200 import simuli as SM, synth  # noqa: E402


def lidar(cfg, scene, **kw):
    r = SM.LidarRenderer(cfg, SM.to_device_scene(scene), **kw)
    r.want_counters(True)
    r.requires_grad(True)
    out = r.scan(sync_capacity=True)
    g = r.backward({"depth": torch.ones_like(out["depth"]), "intensity": torch.ones_like(out["intensity"]),
                    "opacity": torch.ones_like(out["opacity"])})
    torch.cuda.synchronize()
    return int(r.n_pairs.item()), {k: float(v.abs().max()) for k, v in g.items()}


def main():
    quick = "--quick" in sys.argv
    SM.load()
    cfgA, sA = synth.lidar_config("A"), synth.scene_for("A")
    print("A exact", lidar(cfgA, sA), flush=True)
    print("A sat", lidar(cfgA, sA, enable_culling=1), flush=True)
    if not quick:
        cfgB = synth.lidar_config("B")
        sB = synth.scene_for("B", n=200_000)
        print("B-sub", lidar(cfgB, sB), flush=True)
        cfgD = synth.lidar_config("B")
        cfgD.beam_divergence = 1.5e-3
        print("B-sub div", lidar(cfgD, sB), flush=True)
        print("B-sub pray", lidar(cfgB, sB, per_ray_sh=True), flush=True)
    sc = synth.with_actors(sA, seed=3, n_actors=4, per_actor=200)
    print("A actors", lidar(cfgA, sc), flush=True)
    cam = synth.camera_config("D-small")
    cs = synth.corridor_scene(7, 5000 if quick else 20000, x_range=(0.0, 40.0), kind="camera", ego=(1.5, 0.0, 1.6))
    c = SM.CameraRenderer(cam, SM.to_device_scene(cs))
    c.want_counters(True)
    c.requires_grad(True)
    out = c.frame(sync_capacity=True)
    He, We = 16, 32
    env = torch.rand(He, We, 3, device="cuda")
    grid = torch.zeros(4, 8, 8, 12, device="cuda")
    grid[..., 0] = grid[..., 5] = grid[..., 10] = 1.0  # identity 3x4 affine per cell
    comp = c.compose(env, grid)
    g = c.backward({"rgb": torch.ones_like(out["rgb"]), "depth": torch.ones_like(out["depth"])})
    torch.cuda.synchronize()
    print("camera", int(c.n_pairs.item()), float(comp.abs().max()), {k: float(v.abs().max()) for k, v in g.items()},
          flush=True)
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
