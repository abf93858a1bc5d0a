"""Dynamic instructions and stall samples per kernel phase (ncu source page),
phases delimited by the CW_STAMP(k) markers of the profiled cw_frame.cuh.
usage: ncu_phases.py report.ncu-rep [path/to/cw_frame.cuh as built]"""
import csv, re, subprocess, sys
rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_1408_3526_b200/csrc/cw_frame.cuh"
names = {0: "prologue/loop top", 1: "x stage + y SDFT", 2: "TMA wait", 3: "observer+Hz+Hx", 4: "barrier 1",
         5: "C1 Hy/pow/T^", 6: "barrier 2", 7: "CD contraction", 8: "barrier 3", 9: "E pick+PEF",
         10: "barrier 4", 11: "F residual / tail"}
marks = []
for i, line in enumerate(open(src), 1):
    m = re.search(r"CW_STAMP\((\d+)\);", line)
    if m:
        marks.append((i, int(m.group(1))))
def phase(ln):
    p = 11 if ln > marks[-1][0] else None
    prev = None
    for l, k in marks:
        if ln <= l:
            return k if prev is not None or True else 0
        prev = k
    return 11
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
S, E = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
agg = {}
fname = None
for r in rows[hi + 1:]:
    if r and r[0] == "File Path":  # next source file: stop (line numbers collide)
        break
    if not r or not r[0].isdigit() or r[2] != "-":
        continue
    ln = int(r[0])
    if ln < marks[0][0] - 30 or ln > marks[-1][0] + 40:
        k = "other (helpers, prologue)"
    else:
        k = names[phase(ln)]
    s, e = float(r[S] or 0), float(r[E] or 0)
    a = agg.setdefault(k, [0.0, 0.0])
    a[0] += s; a[1] += e
ts = sum(v[0] for v in agg.values()); te = sum(v[1] for v in agg.values())
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} samples {100*s/ts:5.1f}%  instructions {100*e/te:5.1f}%")
