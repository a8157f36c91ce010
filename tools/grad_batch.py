"""Training gradient on a batch of C4 images (default 32): ms per call, MPix/s, and
bitwise reproducibility of two calls.  python tools/grad_batch.py [B]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1510_02930_b200 as P  # noqa: E402
from synth import make_problem  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = make_problem(4)
f = torch.from_numpy(p.f[:B]).cuda()
gt = torch.from_numpy(p.clean[:B]).cuda()
eng = P.TNRD(p.model, device=0)
a = eng.loss_grad(f, gt)
torch.cuda.synchronize()
t0 = time.perf_counter()
b = eng.loss_grad(f, gt)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
same = a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
_, H, W = p.f.shape
print(json.dumps({"B": B, "ms_per_call": dt * 1e3, "MPix_per_s": B * H * W / 1e6 / dt, "bitwise_repeat": bool(same),
                  "engine": "tensor" if eng.engine_for(B, H, W) == P.ENGINE_TENSOR else "fp32"}))
eng.close()
