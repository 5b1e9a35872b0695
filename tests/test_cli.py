"""The command-line harness (paper_2101_09441_b200/cli.py) against the
reference CLI's own outputs on the same files (tests/golden/cli.npz, written
by oracle/gen_golden.py from dblreach's cli.py): build summary and snapshot
bytes, query rows (csv / json / from a snapshot), update streams with exact
per-line insert stats and the saved snapshot.  `visited` of BFS answers is
compared as "== 0 iff label-answered"."""
from __future__ import annotations

import contextlib
import csv
import io
import json

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    d = golden("cli")
    p = tmp_path_factory.mktemp("cli")
    paths = {}
    for key, name in (("graph_txt", "g.txt"), ("queries_txt", "q.txt"), ("updates_txt", "u.txt")):
        paths[key] = str(p / name)
        open(paths[key], "w").write(str(d[key]))
    paths["ref_snapshot"] = str(p / "ref.idx")
    open(paths["ref_snapshot"], "wb").write(d["build_snapshot"].tobytes())
    paths["dir"] = p
    return d, paths


def run(argv):
    from paper_2101_09441_b200 import cli
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def rows_csv(text):
    return list(csv.reader(io.StringIO(text)))


def same_rows(ours, ref):
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert a[:4] == b[:4], (a, b)
        assert (a[4] == "0") == (b[4] == "0"), (a, b)


def test_cli_build_matches_reference(files):
    d, p = files
    snap = str(p["dir"] / "ours.idx")
    rc, out, _ = run(["build", p["graph_txt"], "-o", snap, "--k", "16", "--kprime", "8"])
    assert rc == int(d["build_rc"]) == 0
    ours, ref = json.loads(out), json.loads(str(d["build_out"]))
    for key in ("n", "m", "d_avg", "k", "k_prime", "strategy", "leaves_in", "leaves_out"):
        assert ours[key] == ref[key], key
    assert open(snap, "rb").read() == d["build_snapshot"].tobytes()


@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_cli_query_matches_reference(files, fmt):
    d, p = files
    rc, out, _ = run(["query", p["graph_txt"], p["queries_txt"], "--k", "16", "--kprime", "8", "--format", fmt])
    assert rc == int(d[f"query_{fmt}_rc"]) == 0
    ref = str(d[f"query_{fmt}_out"])
    if fmt == "csv":
        same_rows(rows_csv(out), rows_csv(ref))
    else:
        a = [json.loads(x) for x in out.splitlines()]
        b = [json.loads(x) for x in ref.splitlines()]
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert (x["u"], x["v"], x["reachable"], x["answered_by"]) == (y["u"], y["v"], y["reachable"], y["answered_by"])
            assert (x["visited"] == 0) == (y["visited"] == 0)


def test_cli_query_from_reference_snapshot(files):
    d, p = files
    rc, out, _ = run(["query", p["ref_snapshot"], p["queries_txt"], "--graph", p["graph_txt"]])
    assert rc == 0
    same_rows(rows_csv(out), rows_csv(str(d["query_snap_out"])))


def test_cli_update_stream_exact_stats(files):
    d, p = files
    snap = str(p["dir"] / "upd.idx")
    rc, out, err = run(["update", p["graph_txt"], p["updates_txt"], "--k", "16", "--kprime", "8",
                        "--line-stats", "--save-index", snap])
    assert rc == int(d["update_rc"]) == 0
    ours = [ln for ln in err.splitlines() if ln.startswith("{")]
    ref = [ln for ln in str(d["update_err"]).splitlines() if ln.startswith("{")]
    assert [json.loads(x) for x in ours] == [json.loads(x) for x in ref]
    assert err.splitlines()[-1] == str(d["update_err"]).splitlines()[-1]
    same_rows(rows_csv(out), rows_csv(str(d["update_out"])))
    assert open(snap, "rb").read() == d["update_snapshot"].tobytes()


def test_cli_errors(files):
    d, p = files
    bad = str(p["dir"] / "bad.txt")
    open(bad, "w").write("1 2\n3\n")
    rc, _, err = run(["build", bad])
    assert rc == 1 and "line 2" in err
    dele = str(p["dir"] / "del.txt")
    open(dele, "w").write("- 1000 1007\n")
    rc, _, err = run(["update", p["graph_txt"], dele])
    assert rc == 1 and "deletion" in err
    rc, _, _ = run(["query", p["ref_snapshot"], p["queries_txt"]])
    assert rc == 1   # a snapshot needs --graph
