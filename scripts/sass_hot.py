"""Aggregate an ncu SASS source page (ncu -i X --page source --csv --print-source sass)
per kernel: stall samples and executed instructions by opcode (development aid)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lines = open(path).read().splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
blk = blocks[which]
print(blk[0][:120])
rows = list(csv.reader(blk[1:]))
hdr = rows[0]
iS, iSamp, iNI, iEx = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)"), hdr.index("Instructions Executed")
by = defaultdict(lambda: [0, 0, 0])
tot = [0, 0, 0]
seq = []
for r in rows[1:]:
    if len(r) <= iEx:
        continue
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    try:
        s, ni, ex = float(r[iSamp] or 0), float(r[iNI] or 0), float(r[iEx] or 0)
    except ValueError:
        continue
    by[o][0] += s; by[o][1] += ni; by[o][2] += ex
    tot[0] += s; tot[1] += ni; tot[2] += ex
    seq.append((r[0], r[iS].strip(), s, ex))
print(f"total samples {tot[0]:.0f} not-issued {tot[1]:.0f} executed {tot[2]:.3g}")
for o, v in sorted(by.items(), key=lambda kv: -kv[1][2])[:25]:
    print(f"  {o:10s} exec {v[2]/tot[2]*100:5.1f}%  samples {v[0]/tot[0]*100:5.1f}%  not-issued {v[1]/max(tot[1],1)*100:5.1f}%")
if "--hot" in sys.argv:
    for a, s, smp, ex in sorted(seq, key=lambda t: -t[2])[:40]:
        print(f"{a} {smp:6.0f} {ex:10.0f}  {s}")
