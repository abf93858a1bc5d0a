"""Aggregate ncu source-page samples per CUDA source line (cuda,sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
col = {n: i for i, n in enumerate(hdr)}
S = hdr.index("Warp Stall Sampling (All Samples)")
E = hdr.index("Instructions Executed")
tot_s = tot_e = 0
agg = []
for r in rows[hdr_i + 1:]:
    if r and r[0] == "File Path":  # next source file: stop (line numbers collide)
        break
    if not r or not r[0].isdigit() or r[2] != "-":
        continue
    s, e = float(r[S] or 0), float(r[E] or 0)
    tot_s += s; tot_e += e
    agg.append((s, e, int(r[0]), r[1][:90]))
agg.sort(reverse=True)
print(f"total samples {tot_s:.0f}, warp instr {tot_e:.0f}")
for s, e, ln, src in agg[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/tot_s:5.1f}% samp {100*e/tot_e:5.1f}% inst  L{ln:4d}  {src}")
