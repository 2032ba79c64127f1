"""Ingestion parity (CPU): the loader raises the reference's exceptions with the
reference's messages, re-emits traces exactly as the reference does, and packs
the same SoA columns the golden scenarios carry."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, load_scenario

from paper_2512_08365_b200 import trace_model as tm
from paper_2512_08365_b200.columns import TraceColumns

ERRORS = json.load(open(GOLDEN / "traces" / "errors.json"))


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_errors_match_reference(name):
    case = ERRORS[name]
    if case["exc"] is None:
        tm.parse_trace_lines(case["lines"])
        return
    with pytest.raises(getattr(tm, case["exc"])) as ei:
        tm.parse_trace_lines(case["lines"])
    assert type(ei.value).__name__ == case["exc"]
    assert str(ei.value) == case["msg"]


@pytest.mark.parametrize("preset", ["tf32_misconfig", "join_redundant"])
@pytest.mark.parametrize("side", ["a", "b"])
def test_canonical_reemission_matches_reference(preset, side):
    path = GOLDEN / "traces" / preset / f"trace_{side}.jsonl"
    tr = tm.load_trace(str(path))
    want = (GOLDEN / "traces" / preset / f"trace_{side}.jsonl.canonical").read_text().splitlines()
    assert tm.trace_to_lines(tr) == want


@pytest.mark.parametrize("side", ["a", "b"])
def test_columns_match_golden_scenario(side):
    tr = tm.load_trace(str(GOLDEN / "traces" / "tf32_misconfig" / f"trace_{side}.jsonl"))
    sc = load_scenario("preset_tf32_misconfig")
    cols = TraceColumns.from_trace(tr)
    # the written file orders ops by start; the golden columns follow trace order
    order = np.argsort(sc[f"{side}_op_start"], kind="stable")
    np.testing.assert_array_equal(cols.ts, sc[f"{side}_ts"])
    np.testing.assert_array_equal(cols.watts, sc[f"{side}_watts"])
    np.testing.assert_array_equal(np.sort(cols.op_start), sc[f"{side}_op_start"][order])
    assert cols.signal_span() == tuple(int(x) for x in sc[f"{side}_span"])
    assert cols.ops_sorted


def test_trace_api():
    tr = tm.load_trace(str(GOLDEN / "traces" / "tf32_misconfig" / "trace_a.jsonl"))
    op = tr.operators[0]
    assert tr.operator(op.op_id) is op
    with pytest.raises(KeyError):
        tr.operator("nope")
    assert tr.owner_op(op.kernel_ids[0]) is op
    assert tr.run_count == 2
    lo, hi = tr.span_us()
    assert lo == tr.power[0].timestamp and hi >= tr.power[-1].timestamp
    assert tr.model_input_ids() and tr.model_output_ids()


def test_roundtrip_save(tmp_path):
    tr = tm.load_trace(str(GOLDEN / "traces" / "join_redundant" / "trace_b.jsonl"))
    p = tmp_path / "t.jsonl"
    tm.save_trace(tr, str(p))
    tr2 = tm.load_trace(str(p))
    assert tm.trace_to_lines(tr2) == tm.trace_to_lines(tr)
