"""Attribute ncu warp-stall samples (SASS source page CSV) to CUDA source lines
via nvdisasm line info.  usage: ncu_lines.py <src.csv> <cubin> <mangled-kernel> <source.cu> [kernel-index]"""
import csv, re, subprocess, sys

csvf, cubin, kern, srcf = sys.argv[1:5]
which = int(sys.argv[5]) if len(sys.argv) > 5 else 0
rows = list(csv.reader(open(csvf)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur:
        cur["rows"].append(r)
b = blocks[which]
h = b["hdr"]
i_s, i_a = h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
data = [(int(r[i_s] or 0), int(r[i_a], 16)) for r in b["rows"] if len(r) > i_s]
base = data[0][1]
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
start = out.index(".text." + kern + ":")
body = out[start:].split("\n", 1)[1]
nxt = body.find("\n.text.")
body = body[:nxt] if nxt >= 0 else body
line, amap = None, {}
for l in body.splitlines():
    m = re.search(r"line (\d+)", l)
    if m:
        line = int(m.group(1))
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m2:
        amap[int(m2.group(1), 16)] = line
agg = {}
for s, a in data:
    ln = amap.get(a - base)
    agg[ln] = agg.get(ln, 0) + s
src = open(srcf).read().splitlines()
tot = sum(agg.values())
print(b["name"][:100], "samples", tot)
for ln, s in sorted(agg.items(), key=lambda x: -x[1])[:20]:
    print(f"{s:6d} {100.0 * s / max(tot, 1):5.1f}%  line {ln}: {src[ln - 1].strip()[:90] if ln else ''}")
