"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py REPORT.ncu-rep [--launches launches.csv] --tag r01_m1 \
        --workload hh3d_128x128x128 --nodes 2097152 --alg-bytes 64
Writes profiles/<tag>.md and merges the per-launch DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__inst_executed.sum", "smsp__inst_executed_pipe_fp64.sum",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            d[h] = (r[i], units[i])
        recs.append(d)
    return recs


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def to_bytes(v, unit):
    x = num(v)
    if x is None:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return x * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--nodes", type=int, required=True)
    ap.add_argument("--alg-bytes", type=float, default=64)
    a = ap.parse_args()
    recs = raw(a.report)
    lines = [f"# ncu summary `{a.tag}` — workload {a.workload} ({a.nodes} nodes)", "",
             "Captured with `ncu --set full --clock-control none --import-source on` under gpurun "
             "(one GPU); times are cold-cache and serialised (compare shares, not absolutes).", ""]
    traffic = {}
    for d in recs:
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
        wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
        if rd is not None and wr is not None:
            t = rd + wr
            lines.append(f"| dram bytes / node | {t / a.nodes:.1f} | B (algorithmic {a.alg_bytes}) |")
            traffic.setdefault(name, []).append(t)
        ins = num(d.get("sm__inst_executed.sum", ("", ""))[0])
        if ins:
            lines.append(f"| warp instructions / node | {ins * 32 / a.nodes:.1f} | |")
        fp = num(d.get("smsp__inst_executed_pipe_fp64.sum", ("", ""))[0])
        if fp:
            lines.append(f"| fp64 warp instructions / node | {fp * 32 / a.nodes:.1f} | |")
        lines.append("")
    if a.launches:
        lines.append("## Launch list (`--metrics gpu__time_duration.sum`)")
        lines.append("")
        with open(a.launches) as f:
            txt = f.read()
        body = txt[txt.find('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.DictReader(io.StringIO(body)))
        tot = {}
        for r in rows:
            if r.get("Metric Name") == "gpu__time_duration.sum":
                nm = r["Kernel Name"].split("(")[0]
                tot.setdefault(nm, []).append(num(r["Metric Value"]))
        allt = sum(sum(v) for v in tot.values())
        lines.append("| kernel | launches | total | share |")
        lines.append("|---|---|---|---|")
        for nm, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{nm}` | {len(v)} | {sum(v):.0f} | {sum(v) / allt:.1%} |")
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    cur = {}
    if os.path.exists(tj):
        with open(tj) as f:
            cur = json.load(f)
    per = {k: sum(v) / len(v) for k, v in traffic.items()}
    if per:
        dom = max(per, key=per.get)
        cur[a.workload] = per[dom]
    with open(tj, "w") as f:
        json.dump(cur, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
