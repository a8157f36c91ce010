"""Where the streaming kernel differs from the per-tile kernel (debug): one stage,
small image; prints the rows / columns of the largest differences."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1510_02930_b200 as P
from synth import make_model
rng = np.random.default_rng(7)
H, W, T = int(sys.argv[1]) if len(sys.argv) > 1 else 30, 40, int(sys.argv[2]) if len(sys.argv) > 2 else 1
f = rng.poisson(rng.uniform(0, 4, (1, H, W))).astype(np.float32)
model = make_model(rng, T, 48, 7, 63, float(f.max()))
out = {}
for st in ("1", "0"):
    os.environ["TNRD_STREAM"] = st
    import importlib
    eng = P.TNRD(model)
    u = eng.denoise(torch.from_numpy(f).cuda()); torch.cuda.synchronize()
    out[st] = u.cpu().numpy()[0]; eng.close()
d = np.abs(out["1"] - out["0"])
print("max diff", d.max(), "rows with diff > 1e-3:", np.nonzero(d.max(axis=1) > 1e-3)[0].tolist())
print("cols with diff > 1e-3:", np.nonzero(d.max(axis=0) > 1e-3)[0].tolist())
np.set_printoptions(linewidth=250, precision=1)
print((d > 1e-3).astype(int))
