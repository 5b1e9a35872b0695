"""Build the engine library of another git revision (for same-box A/B timing).

  python tools/build_rev.py HEAD base [DEFINE ...]   # -> paper_2101_09441_b200/_lib/variant_base.so

Run a tool against it with DBL_LIB_PATH=paper_2101_09441_b200/_lib/variant_base.so.
"""
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09441_b200 import build as B  # noqa: E402


def main():
    rev, name, defines = sys.argv[1], sys.argv[2], [f"-D{d}" for d in sys.argv[3:]]
    with tempfile.TemporaryDirectory() as tmp:
        arch = subprocess.run(["git", "-C", B.ROOT, "archive", rev, "paper_2101_09441_b200/csrc", "include"],
                              check=True, capture_output=True).stdout
        subprocess.run(["tar", "-x", "-C", tmp], input=arch, check=True)
        csrc = os.path.join(tmp, "paper_2101_09441_b200", "csrc")
        srcs = [f for f in B.SOURCES if os.path.exists(os.path.join(csrc, f))]
        objs = []
        for src in srcs:
            obj = os.path.join(tmp, src.replace(".cu", ".o"))
            flags = [f if not f.startswith("-I") else "-I" + os.path.join(tmp, "include") for f in B._flags(src)]
            subprocess.check_call([B.NVCC, *B.ARCH, *flags, *defines, "-c", os.path.join(csrc, src), "-o", obj],
                                  stderr=subprocess.DEVNULL)
            objs.append(obj)
        out = os.path.join(B.OUTDIR, f"variant_{name}.so")
        subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, *B.LINK])
        print(out)


if __name__ == "__main__":
    main()
