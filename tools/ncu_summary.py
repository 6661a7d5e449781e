"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py <round-tag> [launches.csv] [report.ncu-rep ...]

Writes profiles/<tag>_launches.md (per-kernel share of the ncu launch list
of the bench command: cold-cache, serialised times, so compare SHARES) and
profiles/<tag>_<report>.md (key metrics of each --set full capture).
"""

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (tcgen05) active %"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "HMMA pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions"),
]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    i_n, i_v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ks = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) <= i_v:
            continue
        name = r[i_n].split("(")[0].replace("void ", "")
        ks[name].append(float(r[i_v].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in ks.values())
    out = [f"# {tag}: ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras` (tools/refresh_profiles.sh)",
           "", "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised:",
           "absolute times are pessimistic; the kernel SHARE of the step is what must agree).", "",
           f"{sum(len(v) for v in ks.values())} launches, {tot / 1e3:.1f} ms total", "",
           "| kernel | launches | mean us | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(ks.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / tot:.3f} |")
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(out) + "\n")


def report(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    base = os.path.basename(path).replace(".ncu-rep", "")
    out = [f"# {tag}: `ncu --set full --clock-control none` capture `{base}`", ""]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append(f"## `{d.get('Kernel Name', '?')[:90]}`")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for key, label in KEYS:
            if key in d:
                out.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
        out.append("")
    with open(os.path.join(PROF, f"{tag}_{base}.md"), "w") as f:
        f.write("\n".join(out) + "\n")
    # per-launch DRAM traffic of each captured kernel, read by bench.py
    tj = os.path.join(PROF, "traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(float(d[k]) * scale.get(u[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        entry = {"dram_bytes_per_launch": tot, "source": f"profiles/{tag}_{base}.md",
                 "duration_us": float(d["gpu__time_duration.sum"])}
        # keyed by kernel and by kernel@capture (several captures of one
        # kernel, e.g. K3 in the headline and in the FREQUENT-heavy regime)
        data[f"{name}@{base}"] = entry
        if base in ("k3_full", "k1k2_full", "k2_full", "diag_full") or name not in data:
            data[name] = entry
    with open(tj, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)


def main(argv):
    tag = argv[0]
    os.makedirs(PROF, exist_ok=True)
    for p in argv[1:]:
        if p.endswith(".csv"):
            launches(p, tag)
        elif p.endswith(".ncu-rep"):
            report(p, tag)


if __name__ == "__main__":
    main(sys.argv[1:])
