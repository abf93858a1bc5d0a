"""Executed warp instructions and stall samples per SASS opcode (ncu source page, sass view)."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and "Source" in r)
hdr = rows[hi]
src = hdr.index("Source")
E = hdr.index("Instructions Executed")
S = hdr.index("Warp Stall Sampling (All Samples)")
ex, sa = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= max(E, S):
        continue
    t = r[src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    try:
        ex[op] += float(r[E] or 0)
        sa[op] += float(r[S] or 0)
    except ValueError:
        pass
te, ts = sum(ex.values()), sum(sa.values())
print(f"total executed {te:.0f}, samples {ts:.0f}")
for op, v in ex.most_common(30):
    print(f"{op:10s} inst {100*v/te:5.1f}%  samples {100*sa[op]/ts:5.1f}%")
