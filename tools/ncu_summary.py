"""Summarise ncu output into profiles/ (run here, after a gpurun profiling job).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel launch count, total and mean duration, share of the captured time, from an
      `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list (cold-cache, serialised).
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic.json [config]]
      key `--set full` metrics per captured kernel (duration, DRAM bytes and throughput, issue
      activity, occupancy, top stall reasons) and, optionally, dram bytes per launch merged into
      traffic.json under "cfg<config>:<kernel>" (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys


def short(name: str) -> str:
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("dc::", "")
    return n


def base(name: str) -> str:  # traffic.json key: no template arguments
    return short(name).split("<")[0]


def launches(csv_path: str, out_md: str):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[hi + 1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        ns = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = ns / 1000.0 if unit in ("ns", "nsecond") else ns if unit in ("us", "usecond") else ns * 1000.0
        k = short(r[ix["Kernel Name"]])
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
        total += us
    lines = [f"# ncu launch list: {os.path.basename(csv_path)}", "",
             "Cold-cache, serialised per-launch durations (`gpu__time_duration.sum`, `--clock-control none`).",
             "Only the kernels' SHARE of the captured time is comparable with the bench's live timers.", "",
             "| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / total:.1f} % |")
    lines.append(f"| **total** | {sum(c for c, _ in agg.values())} | {total:.1f} | | 100 % |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print(out_md)


FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def to_bytes(v: float, unit: str) -> float:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * mult.get(unit, 1)


def full(rep: str, out_md: str, traffic_json: str | None, config: str = "3"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
    stall_cols = stall_cols or [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    lines = [f"# ncu --set full: {os.path.basename(rep)}", ""]
    traffic = {}
    if traffic_json and os.path.exists(traffic_json):
        traffic = json.load(open(traffic_json))
    per_kernel = collections.defaultdict(list)
    for r in data:
        per_kernel[short(r[ix["Kernel Name"]])].append(r)
    for k, rs in per_kernel.items():
        lines += [f"## `{k}` ({len(rs)} launch(es) captured)", "", "| metric | " + " | ".join(f"launch {i}" for i in range(len(rs))) + " |",
                  "|---|" + "---:|" * len(rs)]
        for m, label in FULL_METRICS:
            if m not in ix:
                continue
            vals = [r[ix[m]] for r in rs]
            lines.append(f"| {label} (`{m}`, {units[ix[m]]}) | " + " | ".join(vals) + " |")
        if stall_cols:
            sv = collections.Counter()
            for c in stall_cols:
                try:
                    sv[c] = sum(float(r[ix[c]].replace(",", "")) for r in rs) / len(rs)
                except ValueError:
                    pass
            top = [(c, v) for c, v in sv.most_common(6) if v > 0]
            lines += ["", "Top warp-stall reasons (average over captured launches):", ""]
            for c, v in top:
                lines.append(f"- `{c}`: {v:.2f}")
        try:
            rd = sum(to_bytes(float(r[ix["dram__bytes_read.sum"]].replace(",", "")), units[ix["dram__bytes_read.sum"]]) for r in rs) / len(rs)
            wr = sum(to_bytes(float(r[ix["dram__bytes_write.sum"]].replace(",", "")), units[ix["dram__bytes_write.sum"]]) for r in rs) / len(rs)
            traffic[f"cfg{config}:{base(k)}"] = int(rd + wr)
            lines += ["", f"DRAM traffic per launch (read + write): {int(rd + wr):,} B"]
        except (KeyError, ValueError):
            pass
        lines.append("")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print(out_md)
    if traffic_json:
        json.dump(traffic, open(traffic_json, "w"), indent=1, sort_keys=True)
        print(traffic_json)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None, sys.argv[5] if len(sys.argv) > 5 else "3")
    else:
        raise SystemExit(__doc__)
