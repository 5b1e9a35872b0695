"""Run the reference's own test files (pkg/tests) against this engine.

    python tools/ref_tests.py [--out gpurun_out/ref_tests.json]

Here (where /root/reference exists) it first copies the test files into
baseline/_ref_tests (git-ignored like baseline/_ref, so they travel to the GPU
box with a gpurun snapshot but never enter the repository); on the GPU box it
runs them with tools/dblreach_alias.py, which makes `import dblreach` resolve
to this engine (reference code only for names the engine does not define).
Writes per-test outcomes plus the list of reference names any test used.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "baseline", "_ref_tests")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ref_tests.json"))
    ap.add_argument("--copy-only", action="store_true")
    a = ap.parse_args()
    a.out = os.path.abspath(a.out)
    if os.path.isdir(SRC):
        shutil.rmtree(DST, ignore_errors=True)
        shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__"))
    if a.copy_only:
        return
    if not os.path.isdir(DST):
        sys.exit("baseline/_ref_tests missing: run this once where /root/reference exists")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    xml = a.out + ".junit.xml"
    fb = a.out + ".fallbacks.json"
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.path.join(ROOT, "tools"), DBL_REF_FALLBACKS=fb)
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "dblreach_alias", "-q", "-p", "no:cacheprovider",
                        "--junitxml", xml, "-o", "addopts=", DST], cwd=DST, env=env, capture_output=True, text=True)
    import xml.etree.ElementTree as ET
    tests = []
    for tc in ET.parse(xml).getroot().iter("testcase"):
        status = "passed"
        msg = ""
        for tag in ("failure", "error", "skipped"):
            e = tc.find(tag)
            if e is not None:
                status = {"failure": "failed", "error": "error", "skipped": "skipped"}[tag]
                msg = (e.get("message") or "")[:300]
        tests.append({"test": f"{tc.get('classname')}::{tc.get('name')}", "status": status, "message": msg})
    summary = {s: sum(t["status"] == s for t in tests) for s in ("passed", "failed", "error", "skipped")}
    fallbacks = json.load(open(fb)) if os.path.exists(fb) else []
    json.dump({"summary": summary, "reference_names_used": fallbacks, "tests": tests,
               "pytest_tail": r.stdout[-3000:]}, open(a.out, "w"), indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
