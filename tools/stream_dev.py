"""Streaming-engine development check (GPU): parity of the streaming kernel against
the oracle on small cases and C3, R1 / R2, exact / table, plus the per-tile kernel
for comparison.  Prints one line per case.  python tools/stream_dev.py [quick]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_1510_02930_b200 as P  # noqa: E402
from synth import make_model, make_problem  # noqa: E402


def run(model, f, **kw):
    eng = P.TNRD(model, **kw)
    u = eng.denoise(torch.from_numpy(np.ascontiguousarray(f, np.float32)).cuda())
    torch.cuda.synchronize()
    out = u.cpu().numpy()
    eng.close()
    return out


def case(name, model, f, peak, bc=0, phi=0):
    t = time.time()
    u = run(model, f, boundary=bc, phi_mode=phi)
    worst = 0.0
    for b in range(f.shape[0]):
        ref = oracle.denoise(f[b], model, boundary=bc)
        worst = max(worst, float(np.max(np.abs(u[b] - ref))) / (1e-4 * peak))
    print(f"{name}: margin {worst:.3f} ({time.time() - t:.1f} s)", flush=True)
    return worst


rng = np.random.default_rng(7)
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
shapes = [(1, 30, 40), (2, 67, 131), (1, 129, 59)] if quick else [(1, 30, 40), (2, 67, 131), (1, 129, 59), (1, 7, 300), (3, 200, 64)]
for shp in shapes:
    f = rng.poisson(rng.uniform(0, 4, shp)).astype(np.float32)
    model = make_model(rng, 2, 48, 7, 63, float(max(f.max(), 1.0)))
    for bc in (0, 1):
        case(f"{shp} bc{bc}", model, f, 4.0, bc)
p = make_problem(3)
case("C3", p.model, p.f, float(p.peaks[0]))
if not quick:
    case("C3 R2", p.model, p.f, float(p.peaks[0]), bc=1)
    case("C3 table", p.model, p.f, float(p.peaks[0]), phi=1)
