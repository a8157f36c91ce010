"""Per-image time of the L and S tile configurations vs batch size:
chooses the threshold of choose_tile().  Run once per TNRD_FORCE_TILE value."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1510_02930_b200 as P  # noqa: E402
from synth import make_problem  # noqa: E402

p = make_problem(4, batch=12)
eng = P.TNRD(p.model)
res = {}
for B in (1, 2, 3, 4, 5, 6, 8, 10, 12):
    f = torch.from_numpy(p.f[:B]).cuda()
    u = torch.empty_like(f)
    for _ in range(2):
        P.tnrd_denoise(eng.h, f, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        P.tnrd_denoise(eng.h, f, u)
    e1.record()
    torch.cuda.synchronize()
    res[B] = e0.elapsed_time(e1) / 5
print(json.dumps({"tile": os.environ.get("TNRD_FORCE_TILE"), "ms_per_call_by_batch": res}))
