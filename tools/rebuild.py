"""Rebuild libtnrd.so (product) and optional experiment variants into explibs/.
   python tools/rebuild.py [name:DEF1,DEF2 ...]"""
import importlib.util
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1510_02930_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
t = time.time()
b.build(force=True)
print("product", round(time.time() - t), "s", flush=True)
os.makedirs(os.path.join(ROOT, "explibs"), exist_ok=True)
for arg in sys.argv[1:]:
    name, defs = arg.split(":")
    t = time.time()
    b.build(out=os.path.join(ROOT, "explibs", f"lib_{name}.so"), defines=[d for d in defs.split(",") if d])
    print(name, round(time.time() - t), "s", flush=True)
