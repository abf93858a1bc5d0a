"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
frame-kernel launches and their mean duration vs everything else."""
import csv, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
frame, other = [], collections.Counter()
other_t = 0.0
for r in rows:
    t = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    if "cw_frame_kernel" in r[ki]:
        frame.append(t)
    else:
        other[r[ki][:80]] += 1
        other_t += t
print(f"cw_frame_kernel launches: {len(frame)}, mean {sum(frame)/max(1,len(frame)):.1f} us, "
      f"min {min(frame):.1f}, max {max(frame):.1f}")
print(f"other kernels in the process: {sum(other.values())} launches, {other_t:.1f} us total")
for k, n in other.most_common(8):
    print(f"  {n:6d} x {k}")
