#!/usr/bin/env python
"""Run the reference's own test suite against this build and write a conformance report.

    python conformance/fetch_reference_tests.py      # in the build container (stages tests)
    python conformance/run.py [--out DIR]            # on a GPU box (or here: host-only tests)

Writes DIR/conformance.json (per-test outcome + totals per file) and DIR/conformance.md
(default DIR = gpurun_out/conformance). The shim (conformance/shim/dynsparse) maps every
`dynsparse.*` import onto paper_2502_07590_b200; nothing in the reference tests is edited.
"""

import argparse
import json
import subprocess
import sys
import xml.etree.ElementTree as ET
from collections import Counter, defaultdict
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "conformance"))
    ap.add_argument("pytest_args", nargs="*")
    a = ap.parse_args()
    tests = HERE / "_ref_tests"
    if not tests.is_dir():
        print("conformance/_ref_tests missing: run conformance/fetch_reference_tests.py first")
        return 2
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    xml = out / "junit.xml"
    cmd = [sys.executable, "-m", "pytest", str(tests), "-q", "-p", "no:cacheprovider",
           "--rootdir", str(HERE), "-c", "/dev/null", f"--junitxml={xml}", *a.pytest_args]
    res = subprocess.run(cmd, cwd=str(HERE), capture_output=True, text=True)
    (out / "pytest.log").write_text(res.stdout + "\n" + res.stderr)
    per_file = defaultdict(Counter)
    cases = []
    for tc in ET.parse(xml).getroot().iter("testcase"):
        name = f"{tc.get('classname')}::{tc.get('name')}"
        outcome = "passed"
        msg = ""
        for child in tc:
            if child.tag in ("failure", "error"):
                outcome, msg = "failed", (child.get("message") or "")[:300]
            elif child.tag == "skipped":
                typ = child.get("type") or ""
                outcome = "xfailed" if "xfail" in typ or "xfail" in (child.get("message") or "") else "skipped"
                msg = (child.get("message") or "")[:300]
        parts = tc.get("classname").split(".")
        per_file[next((x for x in parts if x.startswith("test_")), parts[0])][outcome] += 1
        cases.append({"test": name, "outcome": outcome, "message": msg})
    totals = Counter(c["outcome"] for c in cases)
    rep = {"totals": dict(totals), "per_file": {k: dict(v) for k, v in sorted(per_file.items())},
           "cases": cases, "pytest_rc": res.returncode}
    (out / "conformance.json").write_text(json.dumps(rep, indent=1))
    lines = ["# Reference test suite vs this build", "",
             f"Totals: {dict(totals)} (pytest rc {res.returncode})", "",
             "| file | passed | failed | xfailed | skipped |", "|---|---|---|---|---|"]
    for f, c in sorted(per_file.items()):
        lines.append(f"| {f} | {c['passed']} | {c['failed']} | {c['xfailed']} | {c['skipped']} |")
    fails = [c for c in cases if c["outcome"] == "failed"]
    if fails:
        lines += ["", "## Failures", ""] + [f"- `{c['test']}`: {c['message']}" for c in fails]
    (out / "conformance.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:6 + len(per_file) + 2]))
    return 0 if not fails else 1


if __name__ == "__main__":
    sys.exit(main())
