"""Print the hottest SASS lines (stall samples) of an ncu report, with context."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(h) and r[0] != "Address":
        data.append(r)
i_src = h.index("Source"); i_s = h.index("Warp Stall Sampling (All Samples)"); i_ex = h.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
hot = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:n]
mode = sys.argv[3] if len(sys.argv) > 3 else "top"
if mode == "top":
    for k in hot:
        r = data[k]
        print(f"{float(r[i_s] or 0) / tot * 100:5.1f}% {int(float(r[i_ex] or 0)):>10d} {k:5d} {r[i_src][:100]}")
else:
    lo, hi = map(int, mode.split(":"))
    for k in range(lo, hi):
        r = data[k]
        print(f"{float(r[i_s] or 0) / tot * 100:5.1f}% {int(float(r[i_ex] or 0)):>10d} {k:5d} {r[i_src][:100]}")
