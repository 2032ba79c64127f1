"""GPU parity of the tensor-equivalence path (csrc/tensor.cu): batched Jacobi
spectra against the reference's (tests/golden/tensors.json.gz) and the
oracle, exact prefilter norms, and match_tensors against the reference's
pairs, candidate counts and full-check counts."""

import math

import numpy as np
import pytest

from _tensor_cases import data, names, random_tensors, traces
from oracle import tensor_equiv as ot
from paper_2512_08365_b200 import tensor_equiv as te
from paper_2512_08365_b200 import tensor_match as tm

pytestmark = pytest.mark.gpu

SPEC_REL = 1e-11   # singular values: dot products summed in another order than numpy's


def _close(a, b, rel=SPEC_REL):
    assert len(a) == len(b), (a, b)
    for x, y in zip(a, b):
        assert abs(x - y) <= rel * max(abs(x), abs(y)), (x, y)


def test_invariant_sets_match_reference():
    xs = random_tensors()
    got = te.invariant_sets([x for x, _ in xs])
    for (x, want), inv in zip(xs, got):
        assert inv.source_order == x.ndim
        assert len(inv.spectra) == len(want)
        for s, w in zip(inv.spectra, want):
            _close(s.singulars, w)


def test_spectra_match_oracle_on_layout_variants():
    rng = np.random.default_rng(5)
    xs = []
    for shp in [(3, 5, 7), (8, 8), (2, 9, 2, 3), (12, 1, 4), (33, 65), (5, 5, 5, 5)]:
        x = rng.standard_normal(shp)
        xs += [x, np.transpose(x, tuple(reversed(range(x.ndim)))), x.reshape(shp[0], -1)]
    got = te.invariant_sets(xs)
    for x, inv in zip(xs, got):
        want = ot.invariant_set(x)
        for s, w in zip(inv.spectra, want):
            _close(s.singulars, w)


def test_large_unfolding_uses_global_scratch():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((300, 120))  # 36k doubles: beyond the shared-memory tile
    s = te.singular_values(x)
    _close(s.singulars, ot.singular_values(x), 1e-10)
    _close(s.singulars, sorted(np.linalg.svd(x, compute_uv=False), reverse=True), 1e-10)


def test_singular_values_drop_in():
    x = np.arange(12, dtype=np.float64).reshape(3, 4)
    assert len(te.singular_values(x).singulars) == 2  # rank 2, third value trimmed
    _close(te.singular_values(x).singulars, ot.singular_values(x))
    with pytest.raises(ValueError):
        te.singular_values(np.array([[np.nan, 1.0], [1.0, 2.0]]))


def test_norms_bit_exact():
    from paper_2512_08365_b200.tensor_match import _norms
    from paper_2512_08365_b200 import _native
    rng = np.random.default_rng(2)
    segs = [rng.standard_normal(int(n)) * 10.0 ** rng.integers(-8, 8) for n in rng.integers(0, 300, 200)]
    off = np.zeros(len(segs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([s.size for s in segs])
    got = _norms(np.concatenate(segs), off, _native.device()).cpu().numpy()
    assert got.tolist() == [ot.py_norm(s.tolist()) for s in segs]


@pytest.mark.parametrize("name", names())
def test_match_tensors_matches_reference(name):
    ta, tb = traces(name)
    pairs, st = tm.match_tensors(ta, tb)
    g = data()["match"][name]
    assert st.candidate_pairs == g["candidate_pairs"]
    assert st.full_checks == g["full_checks"]
    assert [(p.tensor_a, p.tensor_b) for p in pairs.pairs] == [(a, b) for a, b, _ in g["pairs"]]
    for p, (_, _, s) in zip(pairs.pairs, g["pairs"]):
        assert p.score == pytest.approx(s, rel=1e-6, abs=1e-12)


def test_prefilter_rejections_match_oracle():
    """Norm collisions the reference corpus lacks: equal counts, norms equal or
    just outside epsilon, different spectra."""
    rng = np.random.default_rng(13)
    base = [rng.standard_normal((4, 6)) for _ in range(40)]
    xa = base + [b * (1 + 2e-3) for b in base[:10]]
    xb = [np.roll(b, 1, axis=0) for b in base] + [b.reshape(6, 4) for b in base[10:20]]
    xb += [rng.standard_normal(24) * np.linalg.norm(b) / math.sqrt(24) for b in base[:5]]
    from paper_2512_08365_b200 import _native
    from paper_2512_08365_b200.tensor_match import _norms, _prefilter
    dev = _native.device()

    def pack(xs):
        off = np.zeros(len(xs) + 1, dtype=np.int64)
        off[1:] = np.cumsum([x.size for x in xs])
        return np.concatenate([x.ravel() for x in xs]), off
    va, oa = pack(xa)
    vb, ob = pack(xb)
    na, nb = _norms(va, oa, dev), _norms(vb, ob, dev)
    pa, pb = _prefilter(np.diff(oa), np.diff(ob), na, nb, 1, 1e-3, dev)
    want = ot.prefilter(np.diff(oa).tolist(), np.diff(ob).tolist(), [na.cpu().tolist()], [nb.cpu().tolist()],
                        1e-3)
    assert list(zip(pa.tolist(), pb.tolist())) == want
    # and the full decision on each candidate agrees with the oracle
    for a, b in want:
        eq, s = te.tensors_equivalent(xa[a], xb[b])
        oeq, os_ = ot.equivalent(xa[a], xb[b])
        assert eq == oeq
        if eq:
            assert s == pytest.approx(os_, rel=1e-6, abs=1e-12)


def test_device_embedding_equals_host_restatement():
    """dw_spectra_embed (device) vs embed_injectively (host) on equivalent,
    near-equivalent and unrelated tensor pairs of order 2-4."""
    rng = np.random.default_rng(21)
    xs = []
    for shp in [(3, 4), (2, 3, 4), (4, 4, 5), (2, 2, 3, 3), (6, 5)]:
        x = rng.standard_normal(shp)
        xs += [x, np.transpose(x), x * (1 + 1e-4), x + 1e-3 * rng.standard_normal(shp),
               rng.standard_normal(shp)]
    xs = [x for x in xs if x.ndim > 1]
    vals = np.concatenate([x.ravel() for x in xs])
    offs = np.cumsum([0] + [x.size for x in xs])[:-1]
    b = te.SpectraBatch(vals, [x.shape for x in xs], offs)
    ja, jb = np.meshgrid(np.arange(len(xs)), np.arange(len(xs)), indexing="ij")
    same = np.array([[xs[i].size == xs[j].size for j in range(len(xs))] for i in range(len(xs))])
    ja, jb = ja[same], jb[same]
    for eps in (1e-3, 0.5):
        got = b.embed(ja, jb, eps)
        for g, i, j in zip(got, ja, jb):
            x, y = b.spectra(int(i)), b.spectra(int(j))
            small, large = (x, y) if len(x) <= len(y) else (y, x)
            want = te.embed_injectively(small, large, eps)
            if want is None:
                assert g == math.inf
            else:
                assert g == pytest.approx(want, rel=1e-12, abs=1e-15)


def test_order5_sets_embed_on_host():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 2, 3, 2, 2))
    eq, s = te.tensors_equivalent(x, np.transpose(x, (4, 3, 2, 1, 0)))
    oeq, os_ = ot.equivalent(x, np.transpose(x, (4, 3, 2, 1, 0)))
    assert eq and oeq
    assert s == pytest.approx(os_, abs=1e-12)


def _trace_with(tensors_a, tensors_b):
    """Minimal reference-style traces whose tensors are graph inputs of one op."""
    from paper_2512_08365_b200.trace_model import (OperatorEvent, PowerSample, TensorSnapshot, Trace,
                                                   TraceHeader)

    def mk(tensors):
        snaps = {tid: (TensorSnapshot(tid, tuple(x.shape), tuple(float(v) for v in x.ravel())),)
                 for tid, x in tensors.items()}
        op = OperatorEvent("op0", "f", tuple(sorted(tensors)), (), (), 0, 10)
        return Trace(TraceHeader(1, "s", "w", 0), snaps, (op,), {}, (PowerSample(0, 1.0),), (), None, {})
    return mk(tensors_a), mk(tensors_b)


def test_match_tensors_edge_cases():
    rng = np.random.default_rng(8)
    x = rng.standard_normal((2, 3, 4))
    ta, tb = _trace_with({"a": x, "v": np.arange(5.0)}, {"b": np.transpose(x, (2, 0, 1)), "w": np.arange(5.0)})
    pairs, st = tm.match_tensors(ta, tb)
    assert [(p.tensor_a, p.tensor_b) for p in pairs.pairs] == [("a", "b"), ("v", "w")]
    assert st.candidate_pairs == 2 and st.full_checks == 2
    # no tensors at all
    ea, eb = _trace_with({}, {})
    pairs, st = tm.match_tensors(ea, eb)
    assert len(pairs) == 0 and st.candidate_pairs == 0
    # order above the cap raises once that pair is compared, as the reference does
    big = rng.standard_normal((1,) * 9)
    ba, bb = _trace_with({"a": big}, {"b": big})
    with pytest.raises(ValueError):
        tm.match_tensors(ba, bb)
