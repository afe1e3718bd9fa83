"""Per-region stall breakdown of one kernel from an ncu report's SASS source
page (`ncu -i rep --page source --csv --print-source sass`): the CG loop is
located by its back edge; regions are setup (before the loop), the loop, and
the tail (write-back).  Usage: python scripts/sass_stalls.py sass.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    ins.append((int(r[0], 16), r[1].strip(), r))
base = ins[0][0]
# the CG loop: the last backward branch

def target(t):
    m = re.search(r"BRA[^0-9]*0x([0-9a-f]+)", t)
    return int(m.group(1), 16) if m else None


back = [(a, target(t)) for a, t, _ in ins if target(t) is not None and target(t) < a]
# the CG loop: the backward branch spanning the most code
a1, a0 = max(back, key=lambda b: b[0] - b[1])
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def region(a):
    return "setup" if a < a0 else ("cg loop" if a <= a1 else "tail")


tot = collections.defaultdict(lambda: collections.Counter())
op = collections.defaultdict(lambda: collections.Counter())
inst = collections.Counter()
for a, t, r in ins:
    g = region(a)
    s = int(r[col["# Samples"]] or 0)
    tot[g]["samples"] += s
    inst[g] += int(r[col["Instructions Executed"]] or 0)
    for h in stalls:
        tot[g][h] += int(r[col[h]] or 0)
    name = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
    op[g][name] += s
allsamp = sum(v["samples"] for v in tot.values())
print(f"stall samples by region (share of {allsamp}):")
for g in ("setup", "cg loop", "tail"):
    v = tot[g]
    top = ", ".join(f"{h[6:]} {100 * v[h] / max(v['samples'], 1):.0f}%"
                    for h, _ in sorted(((h, v[h]) for h in stalls), key=lambda kv: -kv[1])[:6])
    print(f"  {g:8s} {100 * v['samples'] / allsamp:5.1f}%  warp-instr {inst[g]:>12d}  [{top}]")
print("samples by opcode in the CG loop:")
lo = op["cg loop"]
s = sum(lo.values())
print("  " + ", ".join(f"{k} {100 * n / s:.1f}%" for k, n in lo.most_common(14)))
