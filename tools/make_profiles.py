"""Summarise ncu captures from gpurun_out/ into tracked files under profiles/.

    python tools/make_profiles.py r1        # reads gpurun_out/prof_r1_k1_{f64,f32}.ncu-rep,
                                            #       gpurun_out/launches_r1.csv
Writes profiles/<tag>_k1_{f64,f32}.txt (key metrics, stall reasons, hot SASS),
profiles/<tag>_launches.txt (per-kernel launch-time shares) and
profiles/k1_traffic.json (dram bytes per K1 launch, read by bench.py).
"""

import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def kernel_summary(rep, tag, dt):
    h, u, v = raw(rep)
    m = {k: (v[i], u[i]) for i, k in enumerate(h)}
    lines = [f"ncu --set full capture of K1 ({dt}), config 2 workload (tools/profile_k1.py --dtype {dt} --L 6)",
             f"kernel: {m.get('Kernel Name', ('?', ''))[0]}", ""]
    for k in KEYS:
        if k in m:
            lines.append(f"  {k:62s} {m[k][0]} {m[k][1]}")
    stalls = {k: float(val) for k, (val, _) in m.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and val.replace(".", "", 1).isdigit()}
    tot = sum(stalls.values()) or 1.0
    lines.append("\n  warp stall samples:")
    for k, val in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
        lines.append(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * val / tot:5.1f}%")
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "12"], capture_output=True,
                         text=True).stdout
    lines.append("\n  hottest SASS (stall share, executions, index, instruction):")
    lines += ["    " + ln for ln in hot.splitlines()]
    with open(os.path.join(PROF, f"{tag}_k1_{dt}.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    return (rd + wr, float(m["gpu__time_duration.sum"][0]), float(m["lts__t_sector_hit_rate.pct"][0]) / 100.0,
            to_bytes(*m["l1tex__m_xbar2l1tex_read_bytes.sum"]))


def launch_summary(path, tag):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = rec["Kernel Name"].split("(")[0]
        unit = rec.get("Metric Unit", "ns")
        val = float(rec["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        per[name][0] += 1
        per[name][1] += val * scale
    tot = sum(t for _, t in per.values()) or 1.0
    lines = [f"ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache serialised launches)",
             f"command: python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e", "",
             f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>7s}"]
    for name, (cnt, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:60]:60s} {cnt:8d} {t:10.3f} {t / cnt:9.4f} {100 * t / tot:6.1f}%")
    with open(os.path.join(PROF, f"{tag}_launches.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    traffic = {}
    for dt in ("f64", "f32"):
        rep = os.path.join(OUT, f"prof_{tag}_k1_{dt}.ncu-rep")
        if os.path.exists(rep):
            b, ms, hit, xbar = kernel_summary(rep, tag, dt)
            traffic[dt] = int(b)
            traffic.setdefault("l2_hit_rate", {})[dt] = round(hit, 4)
            traffic.setdefault("l2_to_sm_bytes", {})[dt] = int(xbar)
    if traffic:
        traffic["source"] = (f"profiles/{tag}_k1_f64.txt, profiles/{tag}_k1_f32.txt "
                             "(ncu --set full, one K1 launch, config 2)")
        with open(os.path.join(PROF, "k1_traffic.json"), "w") as fh:
            json.dump(traffic, fh, indent=1)
    ll = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(ll):
        launch_summary(ll, tag)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
