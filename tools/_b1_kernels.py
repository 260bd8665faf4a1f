"""Per-kernel ncu durations of the last forward pass in a launch list (batch-1 analysis)."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
n = int(sys.argv[2]) if len(sys.argv) > 2 else 14
tot = 0
for r in rows[1:][-n:]:
    tot += float(r[vi]) / 1000
    print(f"{float(r[vi])/1000:8.2f} us  {r[gi] if gi is not None else ''}  {r[ki][:90]}")
print(f"{tot:8.2f} us total")
