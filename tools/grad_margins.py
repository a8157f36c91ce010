"""Measured gradient parity margins: for the test_gpu_grad.py cases, the worst
max|g_gpu - g_oracle| / max|g_oracle| per parameter kind, and its ratio to the test
bound 2e-5.  Prints one JSON object.  python tools/grad_margins.py"""
import json
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1510_02930_b200 as P  # noqa: E402
from synth import make_model  # noqa: E402

CASES = [(2, 24, 20, 2, 4, 3, 15), (1, 33, 40, 3, 6, 5, 31), (1, 40, 36, 2, 8, 7, 63), (1, 96, 80, 8, 48, 7, 63),
         (2, 37, 70, 2, 8, 3, 63), (1, 45, 131, 2, 24, 5, 63), (2, 70, 67, 3, 48, 7, 63)]
if len(sys.argv) > 1:   # one case: B,H,W,T,Nk,k,M
    CASES = [tuple(int(v) for v in sys.argv[1].split(","))]
out = {"bound": 2e-5, "cases": []}
worst = 0.0
for (B, H, W, T, Nk, k, M) in CASES:
    for boundary in (0, 1):
        rng = np.random.default_rng(5 + k + T)
        f = rng.poisson(3.0, size=(B, H, W)).astype(np.float32)
        gt = (f + rng.normal(0, 0.5, size=f.shape)).astype(np.float32)
        m = make_model(rng, T, Nk, k, M, float(f.max()))
        m.rbf_w *= np.float32(3.0)
        eng = P.TNRD(m, boundary=boundary)
        loss, gf, gw, gl = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
        tensor = eng.engine_for(B, H, W) == P.ENGINE_TENSOR
        eng.close()
        rl, rf, rw, rlam = oracle.loss_grad(f, gt, m, boundary)
        rel = {"filters": max(float(np.max(np.abs(np.asarray(gf[t], np.float64) - rf[t])) / np.max(np.abs(rf[t])))
                              for t in range(T)),
               "rbf_w": max(float(np.max(np.abs(np.asarray(gw[t], np.float64) - rw[t])) / np.max(np.abs(rw[t])))
                            for t in range(T)),
               "lambda": float(np.max(np.abs(np.asarray(gl, np.float64) - rlam)) / np.max(np.abs(rlam))),
               "loss": abs(loss - rl) / abs(rl)}
        worst = max(worst, rel["filters"], rel["rbf_w"], rel["lambda"])
        out["cases"].append({"B": B, "H": H, "W": W, "T": T, "Nk": Nk, "k": k, "M": M, "boundary": boundary,
                             "tensor_banks": bool(tensor), "rel_err": rel})
out["worst_rel_err"] = worst
out["worst_fraction_of_bound"] = worst / 2e-5
print(json.dumps(out))
