"""GPU parity of the batched classifier and forced-gap integrals against the
reference (tests/golden/classify.json.gz: detect_waste's categories and
diagnose.forced_gap_joules, run on the reference's presets and fuzz corpus)."""

import numpy as np
import pytest

from _classify_cases import cases, findings, traces
from paper_2512_08365_b200 import diagnose as dg
from paper_2512_08365_b200.columns import TraceColumns
from paper_2512_08365_b200.detect import detect_waste
from paper_2512_08365_b200.energy import build_ledger
from paper_2512_08365_b200.join import join_diff

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(cases()))
def test_categories_match_reference(name):
    ta, tb = traces(name)
    want = [f[4] for f in cases()[name]["findings"]]
    assert dg.classify_findings(findings(name), ta, tb) == want


@pytest.mark.parametrize("name", sorted(cases()))
def test_forced_gap_joules_bit_exact(name):
    ta, tb = traces(name)
    rows = [f for f in cases()[name]["findings"] if f[2] == "waste"]
    for na, nb, _, side, _, want in rows:
        tr, nodes = (ta, na) if side == "A" else (tb, nb)
        assert dg.forced_gap_joules(tr, nodes) == want, (name, nodes)
    # batched: all of a trace's groups in one launch, same values
    for side, tr, k in (("A", ta, 0), ("B", tb, 1)):
        sel = [f for f in rows if f[3] == side]
        if not sel:
            continue
        s = dg._Side(tr)
        got = dg.forced_gap_batch(s, [[s.index_of(o) for o in f[k]] for f in sel])
        assert got == [f[5] for f in sel]


def test_forced_gaps_on_columns_equal_trace_objects():
    name = "tf32_misconfig"
    ta, _ = traces(name)
    ops = [o.op_id for o in ta.operators]
    ca = TraceColumns.from_trace(ta)
    cols = TraceColumns.from_arrays(ca.ts, ca.watts, ca.op_start, ca.op_end, ca.k_start, ca.k_end, ca.k_op,
                                    trace_end=ca.trace_end, op_ids=ops)
    cols.config = dict(ta.config)
    for chunk in (ops[:1], ops[:7], ops[3:40], ops):
        assert dg.forced_gap_joules(cols, chunk) == dg.forced_gap_joules(ta, chunk)


def test_forced_gaps_with_shuffled_kernel_rows():
    """Kernel rows not grouped by owner op take the device sort path."""
    ta, _ = traces("join_redundant")
    ca = TraceColumns.from_trace(ta)
    perm = np.random.default_rng(3).permutation(ca.n_kernels)
    cols = TraceColumns.from_arrays(ca.ts, ca.watts, ca.op_start, ca.op_end, ca.k_start[perm], ca.k_end[perm],
                                    ca.k_op[perm], trace_end=ca.trace_end, op_ids=list(ca.op_ids))
    cols.config = dict(ta.config)
    ops = list(ca.op_ids)
    assert dg.forced_gap_joules(cols, ops) == dg.forced_gap_joules(ta, ops)


@pytest.mark.parametrize("name", ["tf32_misconfig", "fused_api_misuse", "join_redundant"])
def test_detect_waste_classifies_by_default(name):
    ta, tb = traces(name)
    la, lb = build_ledger(ta), build_ledger(tb)
    fs = detect_waste([f.pair for f in findings(name)], la, lb, 0.10, trace_a=ta, trace_b=tb)
    assert [f.category for f in fs] == dg.classify_findings(fs, ta, tb)
    plain = detect_waste([f.pair for f in findings(name)], la, lb, 0.10, trace_a=ta, trace_b=tb,
                         classify=False)
    assert all(f.category == "unknown" for f in plain)
    assert [f.verdict for f in plain] == [f.verdict for f in fs]


def test_join_findings_are_classified():
    ta, tb = traces("join_redundant")
    la, lb = build_ledger(ta), build_ledger(tb)
    jd = join_diff(ta, tb, la, lb, 0.10, 50)
    ca, cb = TraceColumns.from_trace(ta), TraceColumns.from_trace(tb)
    top = jd.top_findings(ca, cb, trace_a=ta, trace_b=tb)
    waste = [f for f in top if f.verdict == "waste"]
    assert waste
    # each join finding classified as the reference classifies that op pair
    want = dg.classify_findings(top, ta, tb)
    assert [f.category for f in top] == want
    # one-sided findings (an operator with no counterpart) are redundant
    for f in waste:
        if not f.pair.nodes_a or not f.pair.nodes_b:
            assert f.category == "redundant"


def test_forced_gaps_without_owner_column():
    """Packed host columns ship no k_op: owners follow from containment in
    sorted, disjoint operators."""
    from paper_2512_08365_b200 import synth
    a, _ = synth.make_pair(synth.scaled(synth.CONFIGS["C4"], 200_000))
    bare = TraceColumns(ts=a.ts, watts=a.watts, trace_end=a.trace_end, op_start=a.op_start, op_end=a.op_end,
                        k_start=a.k_start, k_end=a.k_end)
    ops = list(range(0, a.n_ops, max(1, a.n_ops // 97)))
    want = dg.forced_gap_batch(a, [[o] for o in ops])
    assert dg.forced_gap_batch(bare, [[o] for o in ops]) == want
    q = np.asarray(ops, dtype=np.int64)
    ea, ra = dg._Side(a).kernel_rows(q)
    eb, rb = dg._Side(bare).kernel_rows(q)
    np.testing.assert_array_equal(ea, eb)
    np.testing.assert_array_equal(ra, rb)
    assert ra.size >= len(ops)


def test_kernelless_waste_finding_raises_like_reference():
    """Same op names, no forced gaps, no kernels on either side: the reference's
    analyze_segment_pair raises DiagnoseError (diagnose.py:292-293)."""
    from paper_2512_08365_b200.detect import SubgraphPair, WasteFinding
    from paper_2512_08365_b200.trace_model import OperatorEvent, PowerSample, Trace, TraceHeader

    def mk():
        op = OperatorEvent("o", "matmul", (), (), (), 5, 5)
        return Trace(TraceHeader(1, "s", "w", 0), {}, (op,), {}, (PowerSample(0, 1.0), PowerSample(10, 2.0)),
                     (), None, {})
    ta, tb = mk(), mk()
    f = WasteFinding(pair=SubgraphPair(("o",), ("o",)), energy_a=1.0, energy_b=0.5, energy_ratio=2.0,
                     latency_a=0, latency_b=0, output_rel_diff=0.0, verdict="waste", category="unknown",
                     wasteful_side="A", wasted_joules=0.5, informational=False)
    with pytest.raises(dg.DiagnoseError):
        dg.classify_findings([f], ta, tb)
    # the same pair as columns (no program model): same error
    with pytest.raises(dg.DiagnoseError):
        dg.classify_pairs(TraceColumns.from_trace(ta), TraceColumns.from_trace(tb), ["A"], np.array([0]),
                          np.array([0]))


def test_batched_lcs_alignment_matches_host_rule():
    """csrc/align.cu (one launch for many findings) == the reference's
    table-walk tie rule (diagnose.py:203-224, restated by _lcs_matched) on
    random kernel-name sequences, empty ones included."""
    import random
    from paper_2512_08365_b200.diagnose import _lcs_matched, lcs_matched_batch
    rng = random.Random(5)
    probs = []
    for _ in range(400):
        na, nb = rng.randint(0, 30), rng.randint(0, 30)
        alpha = [f"k{i}" for i in range(rng.randint(1, 6))]
        probs.append(([rng.choice(alpha) for _ in range(na)], [rng.choice(alpha) for _ in range(nb)]))
    got = lcs_matched_batch(probs)
    for (a, b), g in zip(probs, got):
        assert g == _lcs_matched(a, b)
