"""Both tile configurations on every filter size, boundary mode, phi mode and reaction
(DESIGN.md §5.2).  TNRD_FORCE_TILE forces the FP32 engine's large-tile ("L") or
small-tile ("S") kernel (TNRD_ENGINE=fp32) on images small enough for full-image
oracle parity, and the two must agree bitwise (per-pixel arithmetic is independent of
the tiling).  The tensor-core engine is run the same way with two
tile heights (TNRD_TC_ROWS) on the configurations it serves.

Each configuration runs in a subprocess because the override is read once per
process.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from synth import make_model

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1510_02930_b200 as P
from synth import make_model
args = json.loads(sys.argv[2])
rng = np.random.default_rng(args["seed"])
f = rng.poisson(args["peak"] / 2, size=(args["B"], args["H"], args["W"])).astype(np.float32)
m = make_model(rng, args["T"], args["Nk"], args["k"], 63, float(max(f.max(), 1.0)))
eng = P.TNRD(m, boundary=args["bc"], phi_mode=args["phi"], reaction=args["reaction"])
u = eng.denoise(torch.from_numpy(f).cuda()).cpu().numpy()
np.save(args["out"], u)
"""


def _run(tmp_path, tile, engine="fp32", rows=None, **kw):
    out = str(tmp_path / f"u_{tile}_{engine}_{rows}.npy")
    kw["out"] = out
    env = dict(os.environ, TNRD_FORCE_TILE=tile, TNRD_ENGINE=engine)
    if rows:
        env["TNRD_TC_ROWS"] = str(rows)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, json.dumps(kw)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


CASES = [
    dict(k=3, Nk=8, bc=0, phi=0, reaction=0, B=3, H=70, W=93),
    dict(k=5, Nk=24, bc=0, phi=0, reaction=0, B=2, H=65, W=129),
    dict(k=7, Nk=16, bc=1, phi=0, reaction=0, B=2, H=77, W=64),
    dict(k=5, Nk=12, bc=1, phi=1, reaction=0, B=3, H=40, W=72),
    dict(k=7, Nk=12, bc=0, phi=0, reaction=1, B=1, H=130, W=66),
    dict(k=3, Nk=8, bc=0, phi=1, reaction=0, B=5, H=7, W=200),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "k{k}-bc{bc}-phi{phi}-r{reaction}-{B}x{H}x{W}".format(**c))
def test_large_and_small_tiles_match_oracle_and_each_other(tmp_path, case):
    kw = dict(case, T=2, peak=4.0, seed=11)
    uL = _run(tmp_path, "L", **kw)
    uS = _run(tmp_path, "S", **kw)
    assert np.array_equal(uL, uS), "L and S tiles differ"
    rng = np.random.default_rng(11)
    f = rng.poisson(2.0, size=(kw["B"], kw["H"], kw["W"])).astype(np.float32)
    m = make_model(rng, 2, kw["Nk"], kw["k"], 63, float(max(f.max(), 1.0)))
    ref = oracle.denoise(f, m, boundary=kw["bc"], reaction=kw["reaction"])
    err = float(np.max(np.abs(uL - ref)))
    assert err <= 1e-4 * kw["peak"], err


TC_CASES = [
    dict(k=3, Nk=8, bc=0, phi=0, reaction=0, B=3, H=70, W=93),
    dict(k=5, Nk=24, bc=0, phi=0, reaction=0, B=2, H=65, W=129),
    dict(k=7, Nk=48, bc=0, phi=0, reaction=0, B=2, H=77, W=131),
    dict(k=7, Nk=48, bc=0, phi=0, reaction=1, B=1, H=130, W=66),
    dict(k=7, Nk=48, bc=0, phi=0, reaction=0, B=1, H=21, W=200),
    dict(k=7, Nk=48, bc=0, phi=1, reaction=0, B=2, H=40, W=90),
    dict(k=5, Nk=24, bc=0, phi=1, reaction=0, B=1, H=66, W=70),
    dict(k=7, Nk=48, bc=1, phi=0, reaction=0, B=2, H=77, W=131),
    dict(k=7, Nk=48, bc=1, phi=0, reaction=0, B=1, H=7, W=7),
    dict(k=5, Nk=24, bc=1, phi=1, reaction=0, B=1, H=66, W=70),
    dict(k=3, Nk=8, bc=1, phi=0, reaction=0, B=2, H=3, W=40),
]


@pytest.mark.parametrize("case", TC_CASES, ids=lambda c: "tc-k{k}-bc{bc}-phi{phi}-r{reaction}-{B}x{H}x{W}".format(**c))
def test_tensor_engine_tile_heights_match_oracle_and_each_other(tmp_path, case):
    """The tensor-core engine with 16- and 128-row tiles (different M-block and tile
    boundaries) is bitwise equal to itself and within the bar of the oracle."""
    kw = dict(case, T=2, peak=4.0, seed=12)
    u16 = _run(tmp_path, "L", engine="tc", rows=16, **kw)
    u128 = _run(tmp_path, "L", engine="tc", rows=128, **kw)
    assert np.array_equal(u16, u128), "tile heights differ"
    rng = np.random.default_rng(12)
    f = rng.poisson(2.0, size=(kw["B"], kw["H"], kw["W"])).astype(np.float32)
    m = make_model(rng, 2, kw["Nk"], kw["k"], 63, float(max(f.max(), 1.0)))
    ref = oracle.denoise(f, m, boundary=kw["bc"], reaction=kw["reaction"])
    err = float(np.nanmax(np.abs(u16 - ref)))
    assert err <= 1e-4 * kw["peak"], err
