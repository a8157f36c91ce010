"""Print the key numbers of bench.py's JSON line (stdin): label value ms_per_step mean_launch_ms clocks."""
import json
import sys

lines = [l for l in sys.stdin.read().splitlines() if l.startswith("{")]
if not lines:
    print(sys.argv[1] if len(sys.argv) > 1 else "", "NO JSON LINE")
    sys.exit(0)
d = json.loads(lines[-1])
r = d.get("roofline") or {}
print(sys.argv[1] if len(sys.argv) > 1 else "", round(d["value"], 1), d.get("unit"), "ms/step", round(d["ms_per_step"], 4),
      "launch_ms", round(r.get("mean_launch_ms", 0), 4), "frac", round(r.get("frac", 0), 4), "clk", d.get("clocks"))
