"""Hash kernel bandwidth on the c2 primary wave (8.4 M rays): CUDA-event
timed, device-resident inputs; bytes = 24 in + 8 out per ray."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1910_01304_b200 as hb  # noqa: E402
from paper_1910_01304_b200 import scenes  # noqa: E402

sc = scenes.make_scene("c2")
O, D = scenes.primary_rays(sc.camera, sc.spp, seed=0)
Ot, Dt = torch.from_numpy(O).cuda(), torch.from_numpy(D).cuda()
cfg = hb.HashConfig(6)
k = hb.hash_rays(Ot, Dt, cfg)
ref = hb.hash_rays(O, D, cfg)  # staged host path (also GPU)
assert np.array_equal(k.cpu().numpy().view(np.uint64), np.asarray(ref).view(np.uint64))
for _ in range(3):
    hb.hash_rays(Ot, Dt, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    hb.hash_rays(Ot, Dt, cfg)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
n = O.shape[0]
print(f"hash {ms * 1e3:.1f} us per 8.4M-ray wave, {32 * n / ms / 1e6:.0f} GB/s")
