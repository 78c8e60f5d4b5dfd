"""Print the key numbers of a bench.py JSON line read from stdin (or a file)."""
import json
import sys

src = open(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "-" else sys.stdin
tag = sys.argv[2] if len(sys.argv) > 2 else ""
line = [ln for ln in src.read().strip().splitlines() if ln.startswith("{")][-1]
d = json.loads(line)
r = d.get("roofline") or {}
print(tag, "value %.4g" % d["value"], "ms/step %.2f" % d["ms_per_step"],
      "launch %.3f ms" % (r.get("avg_launch_ms") or 0), "frac %.3f" % (r.get("frac") or 0),
      "e2e %s" % (("%.4g" % d["e2e"]["value"]) if d.get("e2e") else None))
print("    host_ms", (d.get("config") or {}).get("host_ms_per_step"))
for k in d.get("kernels_roofline") or []:
    print("   ", k["kernel"], "n=%d" % k["launches"], "%.3f ms" % k["avg_launch_ms"], "frac %.3f" % k["frac"])
if d.get("regrid_stress"):
    s = d["regrid_stress"]
    print("  C5s value %.4g ms/step %.2f" % (s["value"], s["ms_per_step"]))
