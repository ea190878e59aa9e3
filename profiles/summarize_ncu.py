"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python profiles/summarize_ncu.py <tag> [gpurun_out]

Writes profiles/<tag>_launches.md (per-kernel launch count, device time and
share of the step from the `--metrics gpu__time_duration.sum` launch list),
profiles/<tag>_ncu_full.md (key --set full metrics per captured launch) and
profiles/decode_traffic.json (DRAM bytes per decode launch, read by bench.py
as roofline.traffic).
"""
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_uniform.sum", "sm__cycles_elapsed.avg.per_second"]


def short(name):
    m = re.search(r"(\w+_kernel)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:80]


def launches(tag, src):
    path = src / "launches.csv"
    if not path.exists():
        return
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        v = float(r["Metric Value"].replace(",", ""))
        agg[k][1] += v / 1e3 if r["Metric Unit"] == "ns" else (v if r["Metric Unit"] == "us" else v * 1e3)
    total = sum(v[1] for v in agg.values())
    lines = [f"# {tag}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             "Cold-cache, serialised launches: compare shares, not absolute step time.", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.1f} | {t / total:.1%} |")
    (ROOT / "profiles" / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(tag, src):
    reps = sorted(src.glob("prof_*.ncu-rep"))
    out = ["# %s: ncu --set full captures" % tag, ""]
    traffic = None
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        out.append(f"## {rep.name}")
        for r in rows[2:]:
            name = short(r[hdr.index("Kernel Name")])
            grid = r[hdr.index("Grid Size")]
            out.append(f"### `{name}` grid {grid}")
            for k in KEYS:
                if k in hdr:
                    out.append(f"- {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
            if "paged_decode" in name and "dram__bytes_read.sum" in hdr:
                def to_bytes(v, u):
                    v = float(v.replace(",", ""))
                    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
                wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
                traffic = traffic or []
                traffic.append({"kernel": name, "grid": grid, "bytes": rd + wr})
            out.append("")
    (ROOT / "profiles" / f"{tag}_ncu_full.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))
    if traffic:
        # bench.py sums one full + one SWA layer per pair; report mean per launch
        per = sum(t["bytes"] for t in traffic) / len(traffic)
        # the bench line the captured command printed: bench.py only uses this
        # traffic for the exact same workload
        bench = {}
        log = src / "ncu_full_bench.log"
        if log.exists():
            for line in log.read_text().splitlines():
                if line.startswith("{") and '"metric"' in line:
                    bench = json.loads(line)
        (ROOT / "profiles" / "decode_traffic.json").write_text(json.dumps(
            {"source": f"{tag}: ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum",
             "workload": bench.get("config", {}).get("workload"),
             "kernel_launches_per_step": (bench.get("roofline", {}).get("algorithmic_bytes_per_step", 0) //
                                          max(1, bench.get("roofline", {}).get("algorithmic_bytes_per_launch", 1))),
             "algorithmic_bytes_per_launch": bench.get("roofline", {}).get("algorithmic_bytes_per_launch"),
             "launches": traffic, "traffic_bytes_per_launch": per}, indent=1))


def dram(tag, src):
    """Per-kernel achieved DRAM bandwidth from profiles/run_ncu_kernels.sh CSVs:
    one table per workload, grouped by (kernel, grid)."""
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 7672.0
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}
    out = [f"# {tag}: per-kernel DRAM bandwidth (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum --clock-control none)", "",
           "Each launch replayed alone with ncu's cache control (cold L2), so small launches pay their ramp-up;",
           f"GB/s = (DRAM read + write bytes) / device time; % = of the measured copy peak {peak} GB/s.", ""]
    for path in sorted(src.glob("*.csv")):
        rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
        per = defaultdict(dict)
        for r in rows:
            v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
            per[(r["ID"], short(r["Kernel Name"]), r.get("Grid Size", ""))][r["Metric Name"]] = v
        agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
        for (_, k, grid), m in per.items():
            a = agg[(k, grid)]
            a[0] += 1
            a[1] += m.get("gpu__time_duration.sum", 0.0)
            a[2] += m.get("dram__bytes_read.sum", 0.0)
            a[3] += m.get("dram__bytes_write.sum", 0.0)
        if not agg:
            continue
        out += [f"## {path.stem}", "", "| kernel | grid | launches | mean us | read MB | write MB | GB/s | % peak |",
                "|---|---|---|---|---|---|---|---|"]
        for (k, grid), (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            gbs = (rd + wr) / t / 1e9 if t else 0.0
            out.append(f"| `{k}` | {grid} | {n} | {t / n * 1e6:.1f} | {rd / n / 1e6:.1f} | {wr / n / 1e6:.1f} | "
                       f"{gbs:.0f} | {gbs / peak:.1%} |")
        out.append("")
    (ROOT / "profiles" / f"{tag}_kernels_dram.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    if sys.argv[1] == "--dram":
        dram(sys.argv[2], Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "gpurun_out" / "kernels")
        sys.exit(0)
    tag = sys.argv[1]
    src = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out"
    launches(tag, src)
    full(tag, src)
