"""Per-kernel SASS instruction histogram of the built objects (evidence that the hot kernels
are Blackwell-native: tcgen05 MMA / TMEM / TMA / bulk copies; what the gathers and
reductions compile to). python tools/sass_hist.py > profiles/r2/sass_hist.md"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

BUILD = Path(__file__).resolve().parent.parent / "build" / "dsv"
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP",
        "UBLKRED", "LDGSTS", "REDG", "RED", "ATOMG", "ATOMS", "MUFU", "SYNCS", "UCGABAR_ARV",
        "LDS", "STS", "LDG", "STG", "FFMA", "FFMA2", "DFMA", "HMMA"]


def main():
    per = defaultdict(Counter)
    for obj in sorted(BUILD.glob("*.o")):
        out = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
        fn = None
        for line in out.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                fn = m.group(1)
                continue
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
            if fn and m:
                per[(obj.stem, fn)][m.group(2)] += 1
    print("# SASS instruction histogram (sm_100a, `cuobjdump -sass build/dsv/*.o`)\n")
    print("Counts are static instruction counts per kernel (not executions).\n")
    print("| object | kernel | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    names = sorted(per)
    dem = subprocess.run(["c++filt"], input="\n".join(fn for _, fn in names), capture_output=True,
                         text=True).stdout.splitlines()
    for (obj, fn), d in zip(names, dem):
        c = per[(obj, fn)]
        if sum(c.values()) < 50:
            continue
        d = d.split("(")[0]
        name = d if len(d) < 70 else d[:67] + "..."
        print(f"| {obj} | `{name}` | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")


if __name__ == "__main__":
    sys.exit(main())
