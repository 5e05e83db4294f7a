"""Opcode mix of an ncu --page source --print-source sass CSV (executed warp instructions)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
cnt = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iex or not r[iex].strip():
        continue
    n = int(r[iex].replace(",", ""))
    op = r[isrc].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    cnt[o] += n
    tot += n
norm = float(sys.argv[2]) if len(sys.argv) > 2 else tot
print(f"total warp instr {tot}  per unit {tot*32/norm:.1f} thread-instr")
for o, n in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{o:10s} {n*32/norm:8.1f}  {100*n/tot:5.1f}%")
