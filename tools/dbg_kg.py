"""Debug: filter gradient with the tensor-core k-gradient vs the CUDA-core one
(TNRD_GRAD_KG=fp32), error pattern per tap / filter.  python tools/dbg_kg.py [k Nk B H W boundary]"""
import os, subprocess, sys
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "run":
    sys.path.insert(0, "tests"); sys.path.insert(0, ".")
    import torch
    import paper_1510_02930_b200 as P
    from synth import make_model
    k, Nk, B, H, W, bnd = map(int, sys.argv[2:8])
    rng = np.random.default_rng(3)
    f = rng.poisson(3.0, size=(B, H, W)).astype(np.float32)
    gt = (f + rng.normal(0, 0.5, size=f.shape)).astype(np.float32)
    m = make_model(rng, 1, Nk, k, 63, float(f.max()))
    eng = P.TNRD(m, boundary=bnd)
    loss, gf, gw, gl = eng.loss_grad(torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
    np.save(sys.argv[8], np.asarray(gf[0], np.float64))
    sys.exit(0)
args = sys.argv[1:] or ["7", "48", "1", "16", "64", "0"]
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "run", *args, "/tmp/kg_tc.npy"], check=True, env=env)
env["TNRD_GRAD_KG"] = "fp32"
subprocess.run([sys.executable, __file__, "run", *args, "/tmp/kg_ref.npy"], check=True, env=env)
a, b = np.load("/tmp/kg_tc.npy"), np.load("/tmp/kg_ref.npy")
k = int(args[0])
print("shape", a.shape, "max|ref|", np.abs(b).max(), "max err", np.abs(a - b).max())
d = np.abs(a - b).reshape(a.shape[0], k, k)
np.set_printoptions(precision=3, suppress=True, linewidth=150)
print("err per tap (max over filters):\n", d.max(0))
print("err per filter:", d.max((1, 2)))
print("ratio a/b tap-mean filter 0:\n", (a.reshape(-1, k, k)[0] / b.reshape(-1, k, k)[0]))
