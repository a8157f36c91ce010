"""Build experiment variants of libtnrd.so in parallel into explibs/ (the product lib is not rebuilt).
   python tools/pbuild.py name:DEF1,DEF2 ..."""
import importlib.util
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(arg):
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1510_02930_b200", "_build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    name, defs = arg.split(":")
    try:
        b.build(out=os.path.join(ROOT, "explibs", f"lib_{name}.so"), defines=[d for d in defs.split(",") if d])
        return name + " ok"
    except Exception as e:  # noqa: BLE001
        return name + " FAILED " + str(e)


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "explibs"), exist_ok=True)
    with ProcessPoolExecutor(max_workers=8) as ex:
        for r in ex.map(one, sys.argv[1:]):
            print(r, flush=True)
