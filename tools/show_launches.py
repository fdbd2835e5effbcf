"""Prints the per-kernel device times of the last bench step from an ncu launch-list CSV."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[ki].split("(")[0].split("::")[-1][:40], float(r[vi]) / 1e6) for r in rows[hdr + 1:]]
ks = [k for k in ks if "synth" not in k[0]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = len(ks) // steps
tot = 0.0
for name, ms in ks[-n:]:
    print(f"{ms:9.3f} ms  {name}")
    tot += ms
print(f"sum {tot:.3f} ms")
