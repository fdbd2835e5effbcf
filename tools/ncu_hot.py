"""Top stall sites of one kernel in an ncu report, by SASS instruction and (with
a cubin + mangled-name fragment) by source line:
  ncu_hot.py rep.ncu-rep <kernel-index> [n] [cubin mangled-fragment]
Compile with -lineinfo; extract cubins with `cuobjdump -xelf all lib.so`."""
import collections
import csv
import re
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(out.splitlines()):
    if row and row[0] == "Kernel Name":
        cur = [row]
        blocks.append(cur)
    elif cur is not None:
        cur.append(row)
b = blocks[idx]
print(b[0][1][:100])
hdr, data = b[1], [r for r in b[2:] if len(r) > 3]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
samp = lambda r: int(r[iS]) if r[iS].isdigit() else 0
tot = sum(samp(r) for r in data)
print("samples", tot)
for r in sorted(data, key=lambda r: -samp(r))[:n]:
    print(f"{samp(r) / tot * 100:5.1f}% {r[iE]:>10} {r[0][-5:]} {r[1][:90]}")
if len(sys.argv) > 5:
    sass = subprocess.run(["nvdisasm", "-gi", sys.argv[4]], capture_output=True, text=True).stdout
    frag = sys.argv[5]
    lines, on, loc = {}, False, None
    for ln in sass.splitlines():
        if ln.startswith(".text.") or ln.startswith("\t.section"):
            pass
        if re.match(r"^\.text\.\S+:$", ln):
            on = frag in ln
            continue
        if not on:
            continue
        m = re.search(r'## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            loc = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            if m.group(3):
                loc += f" @ {m.group(3).split('/')[-1]}:{m.group(4)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+[^.\s]", ln)
        if m and loc:
            lines[int(m.group(1), 16)] = loc
    base = int(data[0][0], 16)
    agg = collections.Counter()
    reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    why = collections.defaultdict(collections.Counter)
    for r in data:
        key = lines.get(int(r[0], 16) - base, "?")
        agg[key] += samp(r)
        for i in reasons:
            if r[i].isdigit():
                why[key][hdr[i][6:]] += int(r[i])
    print("--- by source line (top stall reasons)")
    for k, v in agg.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else n):
        top = ", ".join(f"{w} {c / max(v, 1) * 100:.0f}%" for w, c in why[k].most_common(3))
        print(f"{v / tot * 100:5.1f}% {k:40s} {top}")
