"""Top instructions of an ncu report by one stall reason (source page, SASS).
    python tools/ncu_hot.py REP [stall_long_sb] [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "# Samples"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
sc, ci = h.index("Source"), h.index(col)
data = []
for k, r in enumerate(rows[2:]):
    if len(r) <= ci:
        continue
    try:
        n = int(r[ci])
    except ValueError:
        continue
    data.append((n, k, r[sc].strip()))
tot = sum(d[0] for d in data) or 1
print(col, "total", tot)
for n, k, s in sorted(data, reverse=True)[:top]:
    print(f"{n / tot * 100:5.2f}% line {k}  {s[:100]}")
