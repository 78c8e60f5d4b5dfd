"""Per-source-line instruction and warp-stall shares of one kernel from an
ncu capture taken with --set full --import-source on.

    ncu -i rep.ncu-rep --page source --csv > src.csv
    cuobjdump -xelf all libmlamr_b200.so && nvdisasm -gi k_step.sm_100a.cubin > k.sass
    python tools/ncu_hot_lines.py k.sass src.csv _ZN5mlamr4wide6k_stepILi2ELb1 [--by inst] [--top 40]

The SASS view of the report and nvdisasm list the kernel's instructions in
the same order; nvdisasm's inline chains give each instruction the line of
csrc/step_tile.cuh it was inlined from (the innermost step_tile.cuh line
below the kernel's own call site)."""
import argparse
import collections
import csv
import os
import re

ap = argparse.ArgumentParser()
ap.add_argument("sass")
ap.add_argument("csv")
ap.add_argument("function")
ap.add_argument("--file", default="step_tile.cuh")
ap.add_argument("--by", default="samples", choices=["samples", "inst"])
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()

sass = open(a.sass).read().split("\n")
start = [i for i, l in enumerate(sass) if l.startswith(".text." + a.function)][0]
end = [i for i, l in enumerate(sass) if l.startswith(".text.") and i > start]
end = end[0] if end else len(sass)
chain, lines, prev = [], [], False
for l in sass[start:end]:
    m = re.search(r'//## File "[^"]*/([^/"]+)", line (\d+)', l)
    if m:
        if not prev:
            chain = []
        chain.append((m.group(1), int(m.group(2))))
        prev = True
        continue
    prev = False
    if re.match(r"\s+/\*[0-9a-f]{4,5}\*/\s+", l):
        lines.append(tuple(chain))
rows = list(csv.reader(open(a.csv)))
hdr, data = rows[1], rows[2:]
assert len(lines) == len(data), (len(lines), len(data))
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for ch, r in zip(lines, data):
    st = [x[1] for x in ch if x[0] == a.file]
    key = st[-2] if len(st) > 1 else (st[-1] if st else 0)
    ie, sp = int(r[ix["Instructions Executed"]]), int(r[ix["# Samples"]])
    agg[key]["inst"] += ie
    agg[key]["samples"] += sp
    tot["inst"] += ie
    tot["samples"] += sp
    for s in stalls:
        agg[key][s] += int(r[ix[s]])
        tot[s] += int(r[ix[s]])
print("warp instructions %d, stall samples %d" % (tot["inst"], tot["samples"]))
print("stalls: " + " ".join("%s %.1f%%" % (s[6:], 100 * tot[s] / tot["samples"])
                            for s in sorted(stalls, key=lambda s: -tot[s])[:10]))
src = []
for root in (os.path.dirname(os.path.abspath(__file__)) + "/../paper_1803_01450_b200/csrc",):
    p = os.path.join(root, a.file)
    if os.path.exists(p):
        src = open(p).read().split("\n")
print("line  inst%  samp%  top stalls (% of all samples) | source")
for k, c in sorted(agg.items(), key=lambda x: -x[1][a.by])[: a.top]:
    top = sorted(((c[s], s[6:]) for s in stalls), reverse=True)[:3]
    print("%4d %5.2f%% %5.2f%% %-44s | %s" % (
        k, 100 * c["inst"] / tot["inst"], 100 * c["samples"] / tot["samples"],
        " ".join("%s:%.1f" % (s, 100 * v / tot["samples"]) for v, s in top),
        src[k - 1].strip()[:72] if 0 < k <= len(src) else ""))
