"""Brief summary of one kernel in an ncu report: time, issue, pipes, stalls,
instruction mix per useful point.   python tools/ncu_brief.py REP [points]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pts = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2]


def g(k):
    return data[hdr.index(k)] if k in hdr else "?"


print(g("Kernel Name")[:80])
for k in ("gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "smsp__inst_executed.sum"):
    print(f"  {k} = {g(k)}")
st = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
        try:
            st.append((float(data[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st) or 1
print("  stalls:", ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie, sc = h.index("Instructions Executed"), h.index("Source")
cnt = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ie or not r[sc].strip():
        continue
    op = r[sc].strip().split()
    o = op[1] if op[0].startswith("@") else op[0]
    try:
        n = int(r[ie] or 0)
    except ValueError:
        continue
    cnt[o.split(".")[0]] += n
    tot += n
scale = 32 / pts if pts else 1 / tot * 100
print(f"  warp-inst {tot}" + (f", thread-inst per point {tot * scale:.1f}" if pts else ""))
print("  " + ", ".join(f"{o} {n * scale:.1f}" for o, n in cnt.most_common(22)))
