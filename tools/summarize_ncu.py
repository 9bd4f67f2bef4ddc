"""Summarise ncu outputs into profiles/ (tracked).

usage: python tools/summarize_ncu.py <tag> <launches.csv> <full.ncu-rep>
Writes profiles/<tag>_launches.md (per-kernel device time share, DRAM bytes per
launch), profiles/<tag>_ncu_full.md (key --set full metrics per kernel) and
profiles/traffic.json (DRAM bytes per launch of each hot kernel from the --set full
capture, else the launch list; read by bench.py as the roofline's `traffic`).
"""

import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name: str) -> str:
    name = name.split("(")[0]
    for pre in ("void ", "dsv::", "attn::", "topk::", "gemm::", "scores::", "simt::"):
        name = name.replace(pre, "")
    return name.strip()


def launches(path: Path, tag: str) -> dict:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
        names[int(r[iid])] = short(r[ik])
    # the timed steps: the last complete step's launches (after the input setup)
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    ours = {k: v for k, v in agg.items() if not k.startswith("at::")}
    total = sum(v[1] for v in agg.values() if True)
    lines = [f"# {tag}: ncu launch list (gpu__time_duration, cold-cache, serialised)", "",
             f"Source: `{path.name}` ({len(per)} launches: input setup + warm-up + 2 timed steps).",
             "Shares are of all listed device time; absolute times are cold-cache and serialised.", "",
             "| kernel | launches | avg time (us) | share of device time | DRAM read / launch (MB) | DRAM write / launch (MB) |",
             "|---|---|---|---|---|---|"]
    for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t / n / 1e3:.1f} | {100 * t / total:.1f}% | {rd / n / 1e6:.1f} | {wr / n / 1e6:.1f} |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    return {k: (v[2] + v[3]) / v[0] for k, v in ours.items()}


def full(path: Path, tag: str) -> dict:
    """Writes the summary; returns DRAM bytes (read + write) per launch of each kernel in the
    --set full capture (the first launch of each name)."""
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    dram = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        try:
            b = sum(float(r[hdr.index(m)].replace(",", "")) * scale.get(units[hdr.index(m)], 1)
                    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        except ValueError:
            continue
        dram.setdefault(short(r[hdr.index("Kernel Name")]), b)
    lines = [f"# {tag}: ncu --set full summary", "",
             f"Source: `{path.name}` (one launch per kernel at the c2 shape, `tools/prof_c2.py`).", ""]
    for r in rows[2:]:
        lines.append(f"## `{short(r[hdr.index('Kernel Name')])}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        lines.append("")
    (PROF / f"{tag}_ncu_full.md").write_text("\n".join(lines))
    return dram


def main():
    tag, lcsv, rep = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
    PROF.mkdir(exist_ok=True)
    traffic = launches(lcsv, tag)
    # per-launch DRAM traffic: the --set full capture where it has the kernel, else the list
    traffic.update(full(rep, tag))
    tj = {k: int(v) for k, v in traffic.items()}
    # bench.py looks kernels up by base name
    for k in list(tj):
        base = k.split("<")[0] if not k.startswith("<") else k
        if base:
            tj.setdefault(base, tj[k])
    (PROF / "traffic.json").write_text(json.dumps(tj, indent=1, sort_keys=True) + "\n")
    print("wrote", PROF)


if __name__ == "__main__":
    main()
