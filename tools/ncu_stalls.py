"""Per-source-line stall breakdown from an ncu report (cuda,sass view)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
reasons = sys.argv[2].split(",") if len(sys.argv) > 2 else ["stall_long_sb", "stall_barrier", "stall_wait", "stall_short_sb", "stall_mio", "stall_no_inst"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
cols = {n: hdr.index(n) for n in reasons}
tot = collections.Counter(); per = {n: collections.Counter() for n in reasons}; src = {}
for r in rows[hi + 1:]:
    if r and r[0] == "File Path":  # next source file: stop (line numbers collide)
        break
    if not r or not r[0].isdigit() or r[2] != "-":
        continue
    ln = int(r[0]); src[ln] = r[1][:80]
    for n, c in cols.items():
        v = float(r[c] or 0); per[n][ln] += v; tot[n] += v
for n in reasons:
    print(f"== {n}: {tot[n]:.0f} samples")
    for ln, v in per[n].most_common(6):
        print(f"   {100*v/max(1,tot[n]):5.1f}%  L{ln:4d} {src[ln]}")
