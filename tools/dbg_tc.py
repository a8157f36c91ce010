import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1510_02930_b200 as P
from synth import make_problem
p = make_problem(3)
f = torch.from_numpy(p.f).cuda()
out = {}
for e in (P.ENGINE_FP32, P.ENGINE_TENSOR):
    eng = P.TNRD(p.model, engine=e)
    out[e] = eng.denoise(f).cpu().numpy()[0]
    eng.close()
d = np.abs(out[1] - out[2])
print('max', d.max(), 'mean', d.mean(), 'nan', np.isnan(out[2]).sum())
ys, xs = np.where(d > 1e-4)
print('bad count', len(ys))
if len(ys):
    print('rows', np.unique(ys)[:20], 'cols', np.unique(xs)[:20])
    print('row hist mod 32', np.bincount(ys % 32, minlength=32))
    print('col hist mod 58', np.bincount(xs % 58, minlength=58))
# single stage model
from synth import Model
m = p.model
m1 = Model(m.filters[:1], m.rbf_w[:1], m.rbf_mu0[:1], m.rbf_step[:1], m.rbf_gamma[:1], m.lam[:1])
o = {}
for e in (P.ENGINE_FP32, P.ENGINE_TENSOR):
    eng = P.TNRD(m1, engine=e)
    o[e] = eng.denoise(f).cpu().numpy()[0]
    eng.close()
d = np.abs(o[1] - o[2]); print('T=1 max', d.max())
ys, xs = np.where(d > 1e-5); print('T=1 bad', len(ys))
if len(ys): print('rows', np.unique(ys)[:40]); print('cols', np.unique(xs)[:40])
