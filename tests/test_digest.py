"""The query digest (query.cu, dbl_index_digest): a u32 per vertex from which a
query batch decides most pairs without reading the label records.

CPU: a numpy restatement of the digest and of its decision rule, checked for
soundness against the oracle's answer codes (every pair the digest decides
gets the code the reference's rule order gives, queries.py:102-108).
GPU: the device digest equals the numpy digest of the exported labels, and
it tracks every label change (inserts, rebuilds, imports, growth), so the
codes of batches that read it equal the codes of batches that read the
records and the oracle's.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2101_09441_b200 import workload as W

FAMS = ("dl_in", "dl_out", "bl_in", "bl_out")
UNDECIDED = 0xFF


def fold14(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64)
    f = x | (x >> np.uint64(14)) | (x >> np.uint64(28)) | (x >> np.uint64(42)) | (x >> np.uint64(56))
    return (f & np.uint64(0x3FFF)).astype(np.uint32)


def np_digest(w: dict) -> np.ndarray:
    """bit 0/1: dl_out has landmark 0 / another landmark; 2/3: same for dl_in;
    4..17 / 18..31: bl_in / bl_out folded onto (bucket % 64) % 14."""
    n = w["bl_in"].shape[0]
    d = np.zeros(n, np.uint32)
    if w["dl_in"].shape[1]:
        for f, sh in (("dl_out", 0), ("dl_in", 2)):
            a = w[f].astype(np.uint64)
            first = (a[:, 0] & np.uint64(1)).astype(np.uint32)
            rest = (a[:, 0] & ~np.uint64(1)) | np.bitwise_or.reduce(a[:, 1:], axis=1) if a.shape[1] > 1 \
                else a[:, 0] & ~np.uint64(1)
            d |= (first | ((rest != 0).astype(np.uint32) << np.uint32(1))) << np.uint32(sh)
    for f, sh in (("bl_in", 4), ("bl_out", 18)):
        fo = np.zeros(n, np.uint32)
        for k in range(w[f].shape[1]):
            fo |= fold14(w[f][:, k])
        d |= fo << np.uint32(sh)
    return d


def np_decide(du: np.ndarray, dv: np.ndarray, use_dl: bool = True, use_bl: bool = True) -> np.ndarray:
    dl = du & (dv >> np.uint32(2)) & np.uint32(3)
    pos = use_dl & ((dl & np.uint32(1)) != 0)
    fi_u, fi_v = (du >> np.uint32(4)) & np.uint32(0x3FFF), (dv >> np.uint32(4)) & np.uint32(0x3FFF)
    blneg = ((fi_u & ~fi_v) | ((dv >> np.uint32(18)) & ~(du >> np.uint32(18)))) != 0
    neg = use_bl & ((not use_dl) | (dl == 0)) & blneg
    out = np.full(len(du), UNDECIDED, np.uint8)
    out[neg] = 2
    out[pos] = 1
    return out


def oracle_case(scale: int, k: int, kp: int, seed: int = 5):
    n = 1 << scale
    src, dst = W.rmat_edges(scale, 8, seed)
    og = O.OracleGraph(n, src, dst)
    oidx = og.build(k, kp, threads=4)
    return n, src, dst, og, oidx


@pytest.mark.parametrize("k,kp", [(64, 64), (256, 64), (0, 64), (100, 200), (64, 1)])
def test_decision_rule_sound_against_oracle(k, kp):
    n, _, _, og, oidx = oracle_case(12, k, kp)
    w = {f: getattr(oidx, f) for f in FAMS}
    dig = np_digest(w)
    rng = np.random.default_rng(11)
    qu = rng.integers(0, n, 200_000, dtype=np.uint32)
    qv = rng.integers(0, n, 200_000, dtype=np.uint32)
    for flags, use_dl, use_bl in ((O.DEFAULT_FLAGS, True, True), (O.DEFAULT_FLAGS & ~O.F_USE_BL, True, False),
                                  (O.DEFAULT_FLAGS & ~O.F_USE_DL, False, True)):
        codes, _ = og.query_batch(oidx, qu, qv, flags=flags, threads=4)
        dec = np_decide(dig[qu], dig[qv], use_dl, use_bl)
        m = (dec != UNDECIDED) & (qu != qv)
        np.testing.assert_array_equal(dec[m], codes[m])
        if use_dl and use_bl and k and kp >= 64:
            assert m.mean() > 0.8, f"digest decided only {m.mean():.3f} of the pairs"


# ------------------------------------------------------------------ GPU --

gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_09441_b200 as E
    return E


@gpu
@pytest.mark.parametrize("k,kp", [(64, 64), (256, 64), (0, 13), (100, 200), (640, 96), (64, 1)])
def test_device_digest_equals_numpy(E, k, kp):
    n = 1 << 12
    src, dst = W.rmat_edges(12, 8, 3)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g, E.IndexConfig(k=k, k_prime=kp))
    np.testing.assert_array_equal(idx.digest(), np_digest(idx.export_words()))


def oracle_codes(g, idx, qu, qv):
    fptr, fcol = g.adjacency(False)
    return O.csr_query_batch(g.vertex_count, fptr.astype(np.uint64), fcol, idx.config.k, idx.config.k_prime,
                             idx.export_words(), qu, qv, threads=4)


@gpu
def test_digest_maintained_through_inserts(E):
    """Batch inserts recompute the changed vertices' digests, single inserts OR
    the new label bits' digest bits in: the digest stays current and exact."""
    scale = 14
    n = 1 << scale
    src, dst = W.rmat_edges(scale, 8, 9)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    rng = np.random.default_rng(4)
    qu = rng.integers(0, n, 20_000, dtype=np.uint32)
    qv = rng.integers(0, n, 20_000, dtype=np.uint32)

    def check(tag):
        dig, current = idx.digest(with_state=True)
        assert current, f"{tag}: digest went stale"
        np.testing.assert_array_equal(dig, np_digest(idx.export_words()), err_msg=tag)
        codes, _ = E.query_codes(g, idx, qu, qv)
        np.testing.assert_array_equal(codes, oracle_codes(g, idx, qu, qv), err_msg=tag)

    check("build")
    for b in range(3):
        iu = rng.integers(0, n, 3000, dtype=np.uint32)
        iv = rng.integers(0, n, 3000, dtype=np.uint32)
        E.insert_edges(g, idx, iu, iv)
        check(f"batch {b}")
    changed = 0
    for _ in range(40):
        changed += E.insert_edge(g, idx, int(rng.integers(0, n)), int(rng.integers(0, n))).labels_changed
    assert changed > 0
    check("single inserts")
    # a hub-to-hub edge: its cones outgrow the single-edge kernel's tables
    # (fallback to the batch fixpoint + change-bitmap refresh)
    E.insert_edge(g, idx, int(n - 1), 0)
    E.insert_edge(g, idx, 1, int(n - 2))
    check("large cones")
    E.rebuild_in_place(g, idx)
    check("rebuild")


@gpu
def test_stale_digest_takes_the_record_path(E):
    """Label writes other than inserts (snapshot import, growth) leave the
    digest stale: small batches read the records, a batch of >= 64k pairs
    recomputes it first."""
    from paper_2101_09441_b200 import snapshot
    import io
    n = 1 << 13
    src, dst = W.rmat_edges(13, 8, 21)
    g = E.DynamicGraph.from_edges(n, src, dst)
    idx = E.build_index(g)
    d0 = idx.digest()
    rng = np.random.default_rng(8)
    qu = rng.integers(0, n, 1 << 17, dtype=np.uint32)
    qv = rng.integers(0, n, 1 << 17, dtype=np.uint32)
    ref = oracle_codes(g, idx, qu, qv)
    buf = io.BytesIO()
    snapshot.save_index(idx, buf)
    buf.seek(0)
    idx2 = snapshot.load_index(buf, g)
    small, _ = E.query_codes(g, idx2, qu[:5000], qv[:5000])
    np.testing.assert_array_equal(small, ref[:5000])
    large, _ = E.query_codes(g, idx2, qu, qv)      # recomputes the digest
    np.testing.assert_array_equal(large, ref)
    dig, current = idx2.digest(with_state=True)
    assert current
    np.testing.assert_array_equal(dig, d0)
    # growth: the new vertex's record is written by insert_vertex
    E.insert_vertex(g, idx, out_edges=[0], in_edges=[1])
    np.testing.assert_array_equal(idx.digest(), np_digest(idx.export_words()))
