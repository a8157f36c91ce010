"""Oracle (double-precision CPU) timing on C1-C3 full images, single-threaded and on all
host cores, next to the paper's own Table II run times (context only: P l.523-540,
single-threaded Matlab on an Intel X5675 and a GTX 780 Ti, l.906-907).  Test
infrastructure: runs the oracle, never the product.

    python tools/oracle_timing.py > profiles/r02_oracle_timing.json
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
import oracle
from synth import make_problem
cfg = int(sys.argv[2])
p = make_problem(cfg)
oracle.lib()
t = time.perf_counter()
oracle.denoise(p.f[0], p.model)
dt = time.perf_counter() - t
print(json.dumps({"seconds": dt, "threads": oracle.num_threads()}))
"""
PAPER = {  # Table II (P l.531-532), seconds; TRDPD_{5x5}^8 / TRDPD_{7x7}^8, CPU (GPU)
    "256x256": {"TRDPD_5x5^8": [1.03, 0.01], "TRDPD_7x7^8": [2.43, 0.02]},
    "512x512": {"TRDPD_5x5^8": [3.07, 0.03], "TRDPD_7x7^8": [7.45, 0.07]},
}


def main():
    out = {"note": "oracle = plain double-precision C (OpenMP over rows); context only, not a target",
           "paper_table_II_seconds_cpu_gpu": PAPER,
           "paper_hardware": "Intel X5675 3.07 GHz single-threaded Matlab; NVIDIA GTX 780 Ti (P l.536-538)",
           "host_cpu": subprocess.run("lscpu | grep 'Model name' | head -1", shell=True, capture_output=True,
                                      text=True).stdout.strip(),
           "nproc": os.cpu_count(), "runs": []}
    for threads in (1, os.cpu_count() or 1):
        for cfg in (1, 2, 3):
            env = dict(os.environ, OMP_NUM_THREADS=str(threads))
            r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(cfg)], env=env, capture_output=True,
                               text=True, timeout=3600)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            sys.path.insert(0, ROOT)
            from synth.generator import CONFIGS
            c = CONFIGS[cfg]
            px = c["H"] * c["W"]
            d.update(config=f"C{cfg}", shape=f"{c['H']}x{c['W']}", T=c["T"], Nk=c["Nk"], k=c["k"],
                     mpix_per_s=px / 1e6 / d["seconds"])
            out["runs"].append(d)
            print(json.dumps(d), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
