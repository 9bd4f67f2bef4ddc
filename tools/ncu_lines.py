"""Per-source-line instruction and warp-stall shares from an ncu report's source page:
python tools/ncu_lines.py report.ncu-rep [top] [kernel-name regex] [launch index]"""
import csv
import subprocess
import sys

cmd = ["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
if len(sys.argv) > 4:
    cmd += ["--launch-skip", sys.argv[4], "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = [r for r in csv.reader(out.splitlines()) if r and r[0].isdigit()]
num = lambda x: int(x) if x.isdigit() else 0   # noqa: E731
# source rows: line, source, '-', '-', stall samples (all), (not issued), samples, instructions
tot_i = sum(num(r[7]) for r in rows) or 1
tot_s = sum(num(r[4]) for r in rows) or 1
print(f"instructions {tot_i}, stall samples {tot_s}")
for r in sorted(rows, key=lambda r: -num(r[4]))[:top]:
    print(f"{int(r[0]):5d}  inst {100 * num(r[7]) / tot_i:5.1f}%  stall {100 * num(r[4]) / tot_s:5.1f}%  {r[1].strip()[:80]}")
