"""Generate golden vectors by running the reference itself.

TEST INFRASTRUCTURE ONLY.  Run in the authoring container (where
/root/reference exists):

    python oracle/gen_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
(and the worked-example tables from its tests/conftest.py), runs it, and
writes small fixtures to tests/golden/.  Nothing here is copied from the
reference: the fixtures are the reference's OUTPUTS on seeded inputs.
The GPU box never needs /root/reference; the tests read only the .npz files.

Fixtures:
  toy.npz        worked example (pkg/tests/conftest.py:15-57): labels from the
                 reference build, the conftest EXPECTED_* tables, all-pairs
                 query codes/visited under several flag sets, the (v9, v2)
                 insertion example (tests/test_updates.py:19-65).
  leaf_hash.npz  leaf_hash KATs (labels.py:119-137) over ids x k' x seeds.
  landmarks.npz  select_landmarks for every strategy on seeded graphs.
  family.npz     C4-style family (tests/test_acceptance.py:30-37): graphs,
                 metadata, labels, all-pairs codes, insert-sequence results.
  cfg1.npz       BASELINE config 1 (ER 10k/50k, 100k queries, 1000 inserts).
  cli.npz        the reference CLI (cli.py) on small files: build summary and
                 snapshot bytes, query output (csv, json, from a snapshot),
                 an update stream with per-line stats and the saved snapshot.
  label_tests.npz  dl_intersec / bl_contain (labels.py:315-327) for all pairs
                 of the worked example (the KATs of tests/test_labels.py:166-191
                 are rows of it) and of seeded random graphs with one- and
                 multi-word labels, with those graphs' reference labels.

    python oracle/gen_golden.py [fixture ...]     # default: all fixtures
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
import dblreach as R  # noqa: E402
import conftest as RC  # noqa: E402  (reference worked-example tables)

ANS = [a.value for a in R.AnsweredBy]
FLAGSETS = {
    "default": R.QueryFlags(),
    "dl_only": R.QueryFlags(use_bl=False),
    "bl_only": R.QueryFlags(use_dl=False),
    "no_early": R.QueryFlags(use_thm1=False, use_thm2=False),
    "no_prune": R.QueryFlags(prune_dl=False, prune_bl=False),
    "bare": R.QueryFlags(use_thm1=False, use_thm2=False, prune_dl=False, prune_bl=False),
}


def flag_bits(f) -> int:
    return (int(f.use_dl) | int(f.use_bl) << 1 | int(f.use_thm1) << 2 | int(f.use_thm2) << 3
            | int(f.prune_dl) << 4 | int(f.prune_bl) << 5)


def words(masks, width):
    w = max(1, (width + 63) // 64) if width else 0
    out = np.zeros((len(masks), w), np.uint64)
    for i, m in enumerate(masks):
        for j in range(w):
            out[i, j] = (m >> (64 * j)) & ((1 << 64) - 1)
    return out


def edges_of(g):
    e = list(g.edges())
    return (np.array([u for u, _ in e], np.uint32), np.array([v for _, v in e], np.uint32))


def index_arrays(prefix, g, idx):
    n = g.vertex_count
    flags = np.zeros(n, np.uint8)
    bucket = np.zeros(n, np.uint32)
    for v in idx.leaf_sets.leaves_in:
        flags[v] |= 1
    for v in idx.leaf_sets.leaves_out:
        flags[v] |= 2
    for v, b in idx.leaf_sets.bucket.items():
        bucket[v] = b
    return {
        f"{prefix}landmarks": np.array(idx.landmark_set.landmarks, np.uint32),
        f"{prefix}leaf_flags": flags,
        f"{prefix}bucket": bucket,
        f"{prefix}dl_in": words(idx.dl_in, idx.config.k),
        f"{prefix}dl_out": words(idx.dl_out, idx.config.k),
        f"{prefix}bl_in": words(idx.bl_in, idx.config.k_prime),
        f"{prefix}bl_out": words(idx.bl_out, idx.config.k_prime),
    }


def outcomes_arrays(outs):
    codes = np.array([ANS.index(o.answered_by.value) for o in outs], np.uint8)
    reach = np.array([o.reachable for o in outs], np.bool_)
    visited = np.array([o.visited for o in outs], np.uint32)
    return codes, reach, visited


def gen_toy():
    g = RC.example_graph()
    idx = RC.example_index(g)
    d = {"n": np.int64(11), "k": np.int64(2), "k_prime": np.int64(2)}
    d["src"], d["dst"] = edges_of(g)
    d.update(index_arrays("", g, idx))
    for name, table in (("exp_dl_in", RC.EXPECTED_DL_IN), ("exp_dl_out", RC.EXPECTED_DL_OUT),
                        ("exp_bl_in", RC.EXPECTED_BL_IN), ("exp_bl_out", RC.EXPECTED_BL_OUT)):
        d[name] = np.array([sum(1 << b for b in table[v]) for v in range(11)], np.uint64)
    pairs = [(u, v) for u in range(11) for v in range(11)]
    d["qu"] = np.array([p[0] for p in pairs], np.uint32)
    d["qv"] = np.array([p[1] for p in pairs], np.uint32)
    for name, fl in FLAGSETS.items():
        outs = [R.query(g, idx, u, v, fl) for u, v in pairs]
        d[f"codes_{name}"], d[f"reach_{name}"], d[f"visited_{name}"] = outcomes_arrays(outs)
        d[f"flagbits_{name}"] = np.int64(flag_bits(fl))
    # insertion example (tests/test_updates.py:19-65): insert (v9, v2)
    g2 = RC.example_graph()
    idx2 = RC.example_index(g2)
    st = R.insert_edge(g2, idx2, RC.V9, RC.V2)
    d["ins_uv"] = np.array([RC.V9, RC.V2], np.uint32)
    d["ins_stats"] = np.array([st.visited, st.labels_changed, st.early_terminated], np.uint32)
    d.update(index_arrays("ins_", g2, idx2))
    # certified edge (v2, v5): early terminated
    g3 = RC.example_graph()
    idx3 = RC.example_index(g3)
    st3 = R.insert_edge(g3, idx3, RC.V2, RC.V5)
    d["ins2_uv"] = np.array([RC.V2, RC.V5], np.uint32)
    d["ins2_stats"] = np.array([st3.visited, st3.labels_changed, st3.early_terminated], np.uint32)
    # default-config (selected metadata) build of the toy graph, k = 3
    idx4 = R.build_index(g, R.IndexConfig(k=3, k_prime=4))
    d.update(index_arrays("auto_", g, idx4))
    return d


def gen_leaf_hash():
    rng = np.random.default_rng(7)
    ids = np.concatenate([np.arange(0, 64), rng.integers(0, 2**32, 1000, dtype=np.uint64)])
    kps = np.array([1, 2, 3, 13, 64, 96, 1000], np.uint32)
    seeds = np.array([0, 1, 7, 12345, 2**40 + 3], np.uint64)
    out = np.zeros((len(ids), len(kps), len(seeds)), np.uint32)
    for i, v in enumerate(ids):
        for j, kp in enumerate(kps):
            for s, sd in enumerate(seeds):
                out[i, j, s] = R.leaf_hash(int(v), int(kp), int(sd))
    return {"ids": ids.astype(np.uint64), "kprimes": kps, "seeds": seeds, "buckets": out}


def gen_landmarks():
    d = {}
    cases = [(40, 3, 1, False), (120, 6, 2, True), (300, 2, 3, False), (500, 10, 4, False)]
    for ci, (n, deg, seed, acyc) in enumerate(cases):
        g = R.gen_random_graph(n, deg, seed, acyclic=acyc)
        d[f"c{ci}_n"] = np.int64(n)
        d[f"c{ci}_src"], d[f"c{ci}_dst"] = edges_of(g)
        for s in R.LandmarkStrategy:
            k = min(32, n)
            d[f"c{ci}_{s.value}"] = np.array(R.select_landmarks(g, k, s).landmarks, np.uint32)
        for thr in (0, 2, 6):
            ls = R.select_leaves(g, thr, k_prime=13, hash_seed=5)
            flags = np.zeros(n, np.uint8)
            bucket = np.zeros(n, np.uint32)
            for v in ls.leaves_in:
                flags[v] |= 1
            for v in ls.leaves_out:
                flags[v] |= 2
            for v, b in ls.bucket.items():
                bucket[v] = b
            d[f"c{ci}_leaf_flags_t{thr}"] = flags
            d[f"c{ci}_bucket_t{thr}"] = bucket
    return d


DEGREES = [1, 2, 4, 8, 12, 20]


def gen_family(count=14):
    """A subset of the acceptance family (tests/test_acceptance.py:30-37)."""
    d = {"count": np.int64(count)}
    for i in range(count):
        n = 20 + (i * 173) % 181
        acyclic = i % 2 == 1
        degree = DEGREES[i % len(DEGREES)]
        k = 8 if (n < 64 or i % 3 == 0) else 64
        g = R.gen_random_graph(n, degree, seed=1000 + i, acyclic=acyclic)
        idx = R.build_index(g, R.IndexConfig(k=k, k_prime=k))
        p = f"f{i}_"
        d[p + "n"], d[p + "k"] = np.int64(n), np.int64(k)
        d[p + "src"], d[p + "dst"] = edges_of(g)
        d.update(index_arrays(p, g, idx))
        pairs = [(u, v) for u in range(n) for v in range(n)]
        for name in ("default", "bl_only", "bare"):
            outs, _ = R.query_batch(g, idx, pairs, flags=FLAGSETS[name])
            c, r, vis = outcomes_arrays(outs)
            d[p + f"codes_{name}"] = c
            d[p + f"visited_{name}"] = vis
        # insert sequence (tests/test_acceptance.py:124-139), per-edge stats
        free = n * (n - 1) - g.edge_count
        evs = R.gen_insert_workload(g, min(60, free), seed=2000 + i)
        stats = []
        for ev in evs:
            st = R.insert_edge(g, idx, ev.u, ev.v)
            stats.append((st.visited, st.labels_changed, int(st.early_terminated)))
        d[p + "ins_u"] = np.array([e.u for e in evs], np.uint32)
        d[p + "ins_v"] = np.array([e.v for e in evs], np.uint32)
        d[p + "ins_stats"] = np.array(stats, np.uint32).reshape(-1, 3)
        d.update(index_arrays(p + "after_", g, idx))
        assert idx.labels_equal(R.rebuild_index(g, idx))
    return d


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_cfg1():
    g = R.gen_random_graph(10_000, 5, seed=1)
    idx = R.build_index(g, R.IndexConfig())
    queries = R.gen_random_queries(10_000, 100_000, seed=2)
    outs, stats = R.query_batch(g, idx, queries)
    d = {"n": np.int64(10_000)}
    d["src"], d["dst"] = edges_of(g)
    d.update(index_arrays("", g, idx))
    d["qu"] = np.array([q[0] for q in queries], np.uint32)
    d["qv"] = np.array([q[1] for q in queries], np.uint32)
    d["codes"], _, d["visited"] = outcomes_arrays(outs)
    evs = R.gen_insert_workload(g, 1000, seed=3)
    st = [R.insert_edge(g, idx, e.u, e.v) for e in evs]
    d["ins_u"] = np.array([e.u for e in evs], np.uint32)
    d["ins_v"] = np.array([e.v for e in evs], np.uint32)
    d["ins_stats"] = np.array([(s.visited, s.labels_changed, int(s.early_terminated))
                               for s in st], np.uint32)
    d.update(index_arrays("after_", g, idx))
    return d


def gen_snapshots():
    """Reference save_index bytes (snapshot.py:76-101) for several indexes."""
    import io
    d = {}
    cases = {
        "toy": (RC.example_graph(), None),
        "rand_k13": (R.gen_random_graph(70, 3, seed=5), R.IndexConfig(k=13, k_prime=96, leaf_threshold=2,
                                                                     landmark_strategy=R.LandmarkStrategy.SUM,
                                                                     hash_seed=9)),
        "rand_k64": (R.gen_random_graph(300, 4, seed=6), R.IndexConfig()),
        "rand_k130": (R.gen_random_graph(200, 5, seed=7, acyclic=True), R.IndexConfig(k=130, k_prime=1)),
    }
    for name, (g, cfg) in cases.items():
        idx = RC.example_index(g) if cfg is None else R.build_index(g, cfg)
        buf = io.BytesIO()
        R.save_index(idx, buf)
        d[f"{name}_bytes"] = np.frombuffer(buf.getvalue(), np.uint8)
        d[f"{name}_src"], d[f"{name}_dst"] = edges_of(g)
        d[f"{name}_n"] = np.int64(g.vertex_count)
    return d


def gen_label_tests():
    """dl_intersec / bl_contain of the reference on all pairs."""
    d = {}
    g = RC.example_graph()
    idx = RC.example_index(g)
    pairs = [(x, y) for x in range(11) for y in range(11)]
    d["toy_x"] = np.array([p[0] for p in pairs], np.uint32)
    d["toy_y"] = np.array([p[1] for p in pairs], np.uint32)
    d["toy_dl"] = np.array([R.dl_intersec(idx, x, y) for x, y in pairs], np.uint8)
    d["toy_bl"] = np.array([R.bl_contain(idx, x, y) for x, y in pairs], np.uint8)
    cases = {"r64": (90, 4, 11, R.IndexConfig(k=64, k_prime=64)),
             "r130": (150, 3, 12, R.IndexConfig(k=130, k_prime=96, leaf_threshold=2)),
             "dag": (100, 5, 13, R.IndexConfig(k=20, k_prime=7))}
    for name, (n, deg, seed, cfg) in cases.items():
        g = R.gen_random_graph(n, deg, seed=seed, acyclic=name == "dag")
        idx = R.build_index(g, cfg)
        p = name + "_"
        d[p + "n"], d[p + "k"], d[p + "k_prime"] = np.int64(n), np.int64(cfg.k), np.int64(cfg.k_prime)
        d[p + "threshold"] = np.int64(cfg.leaf_threshold)
        d[p + "src"], d[p + "dst"] = edges_of(g)
        d.update(index_arrays(p, g, idx))
        d[p + "dl"] = np.array([[R.dl_intersec(idx, x, y) for y in range(n)] for x in range(n)], np.uint8)
        d[p + "bl"] = np.array([[R.bl_contain(idx, x, y) for y in range(n)] for x in range(n)], np.uint8)
    return d


def gen_cli():
    """The reference CLI (cli.py) on small files: build summary + snapshot
    bytes, query output (csv and json), an update stream with line stats."""
    import contextlib
    import io
    import tempfile
    from dblreach import cli as RCLI
    d = {}
    rng = np.random.default_rng(5)
    # original ids are sparse and unordered, so the dense remap is exercised
    ids = rng.permutation(np.arange(1000, 1000 + 7 * 60, 7))[:60]
    g = R.gen_random_graph(60, 2.5, seed=9)
    edges = [(int(ids[u]), int(ids[v])) for u, v in g.edges()]
    lines = ["# test graph"] + [f"{u} {v}" for u, v in edges] + [f"{edges[0][0]} {edges[0][1]}"]
    qs = [(int(ids[a]), int(ids[b])) for a, b in rng.integers(0, 60, (300, 2))]
    ups = []
    for a, b in rng.integers(0, 60, (40, 2)):
        ups.append(f"+ {int(ids[a])} {int(ids[b])}")
        if a % 3 == 0:
            ups.append(f"? {int(ids[b])} {int(ids[a])}")
    ups.append("+ 5000 5001")          # unseen ids: new vertices
    ups.append(f"+ {int(ids[0])} 5000")
    ups.append(f"? {int(ids[1])} 5001")
    with tempfile.TemporaryDirectory() as tmp:
        gp, qp, up, sp = (os.path.join(tmp, x) for x in ("g.txt", "q.txt", "u.txt", "s.idx"))
        open(gp, "w").write("\n".join(lines) + "\n")
        open(qp, "w").write("\n".join(f"{a} {b}" for a, b in qs) + "\n")
        open(up, "w").write("\n".join(ups) + "\n")

        def run(argv):
            out, err = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
                rc = RCLI.main(argv)
            return rc, out.getvalue(), err.getvalue()
        rc, out, _ = run(["build", gp, "-o", sp, "--k", "16", "--kprime", "8"])
        d["build_rc"], d["build_out"] = np.int64(rc), np.array(out)
        d["build_snapshot"] = np.frombuffer(open(sp, "rb").read(), np.uint8)
        for fmt in ("csv", "json"):
            rc, out, _ = run(["query", gp, qp, "--k", "16", "--kprime", "8", "--format", fmt, "--workers", "1"])
            d[f"query_{fmt}_rc"], d[f"query_{fmt}_out"] = np.int64(rc), np.array(out)
        rc, out, _ = run(["query", sp, qp, "--graph", gp, "--workers", "1"])
        d["query_snap_rc"], d["query_snap_out"] = np.int64(rc), np.array(out)
        rc, out, err = run(["update", gp, up, "--k", "16", "--kprime", "8", "--line-stats", "--save-index", sp])
        d["update_rc"], d["update_out"], d["update_err"] = np.int64(rc), np.array(out), np.array(err)
        d["update_snapshot"] = np.frombuffer(open(sp, "rb").read(), np.uint8)
        d["graph_txt"], d["queries_txt"], d["updates_txt"] = (np.array(open(p).read()) for p in (gp, qp, up))
    return d


FIXTURES = {"toy": gen_toy, "leaf_hash": gen_leaf_hash, "landmarks": gen_landmarks, "family": gen_family,
            "cfg1": gen_cfg1, "snapshots": gen_snapshots, "label_tests": gen_label_tests, "cli": gen_cli}


def main():
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[1:] or list(FIXTURES)
    for name in names:
        fn = FIXTURES[name]
        d = fn()
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
