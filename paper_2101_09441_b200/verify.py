"""Label verifier (drop-in for the reference's verify_labels).

Reference: updates.py:297-363.  The union-fixpoint check and the optional
exhaustive rebuild comparison run on the GPU (csrc/verify.cu); violations
come back as data (LabelViolation rows sorted by vertex, then family), never
as exceptions.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .graph import as_device_graph
from .labels import DblIndex
from .queries import _check_consistent


@dataclass(frozen=True)
class LabelViolation:
    """One vertex/family pair where the stored label is wrong (updates.py:297-314)."""

    vertex: int
    family: str   # "dl_in" | "dl_out" | "bl_in" | "bl_out"
    expected: int
    actual: int

    def __str__(self) -> str:
        missing = self.expected & ~self.actual
        extra = self.actual & ~self.expected
        bits = lambda x: [i for i in range(x.bit_length()) if x >> i & 1]  # noqa: E731
        parts = []
        if missing:
            parts.append(f"missing bits {bits(missing)}")
        if extra:
            parts.append(f"stale bits {bits(extra)}")
        return f"{self.family}({self.vertex}): {', '.join(parts)}"


@dataclass
class VerifyReport:
    ok: bool
    violations: list[LabelViolation] = field(default_factory=list)


def _int(words) -> int:
    x = 0
    for j, w in enumerate(words):
        x |= int(w) << (64 * j)
    return x


def verify_labels(g, idx: DblIndex, exhaustive: bool | None = None, max_report: int = 100_000) -> VerifyReport:
    """Diagnostic check (updates.py:323-363); exhaustive defaults to n <= 500."""
    g = as_device_graph(g)
    _check_consistent(g, idx)
    if exhaustive is None:
        exhaustive = g.vertex_count <= 500
    H = idx.wdl + idx.wbl
    cnt = ctypes.c_uint64()
    vert = np.zeros(max_report, np.uint32)
    half = np.zeros(max_report, np.uint8)
    exp = np.zeros((max_report, max(H, 1)), np.uint64)
    act = np.zeros((max_report, max(H, 1)), np.uint64)
    N.call("dbl_verify", idx.handle, g.handle, int(bool(exhaustive)), max_report, ctypes.byref(cnt), N.ptr(vert),
           N.ptr(half), N.ptr(exp), N.ptr(act))
    k = min(int(cnt.value), max_report)
    found: dict[tuple[int, str], LabelViolation] = {}
    wdl = idx.wdl
    for i in range(k):
        v, h = int(vert[i]), int(half[i])
        fams = (("dl_in", "bl_in") if h == 0 else ("dl_out", "bl_out"))
        for name, lo, hi in ((fams[0], 0, wdl), (fams[1], wdl, H)):
            e, a = _int(exp[i, lo:hi]), _int(act[i, lo:hi])
            if e != a:
                found[(v, name)] = LabelViolation(v, name, e, a)
    violations = [found[key] for key in sorted(found)]
    return VerifyReport(ok=not violations, violations=violations)
