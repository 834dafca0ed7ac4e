"""Hash of the sorted ids / tile ranges of three config-B poses (compare across
SIMULI_SORT_VARIANT builds: every sweep shape must give the identical stable order)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_12901_b200 import simuli as SM, synth
cfg = synth.lidar_config("B")
r = SM.LidarRenderer(cfg, SM.to_device_scene(synth.scene_for("B")))
h = hashlib.sha256()
for p0, p1 in synth.batch_poses(512)[::200]:
    r.scan(p0, p1, sync_capacity=True)
    torch.cuda.synchronize()
    P = int(r.n_pairs.item())
    h.update(r.sorted_ids[:P].cpu().numpy().tobytes())
    h.update(r.tile_ranges.cpu().numpy().tobytes())
    h.update(r.out["depth"].cpu().numpy().tobytes())
print(os.environ.get("SIMULI_SORT_VARIANT", "default"), h.hexdigest()[:16])
