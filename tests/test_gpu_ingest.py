"""GPU JSONL ingestion (csrc/ingest.cu, ingest.load_columns) vs the
reference-compatible Python loader: the same columns for canonical scale
traces (parsed on the device), the same columns for everything else (taken
by the Python path), and the same exceptions for broken files."""
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

dw = pytest.importorskip("paper_2512_08365_b200")
from paper_2512_08365_b200 import TraceColumns, load_trace  # noqa: E402
from paper_2512_08365_b200.ingest import load_columns  # noqa: E402
from paper_2512_08365_b200.trace_model import (KernelEvent, OperatorEvent, PowerSample, Trace,  # noqa: E402
                                               TraceHeader, trace_to_lines)


def _synthetic_trace(n_ops=3000, seed=0):
    rng = np.random.default_rng(seed)
    ops, kernels, t = [], {}, 10_000
    corr = 0
    for i in range(n_ops):
        nk = int(rng.integers(1, 4))
        kids, s0 = [], t
        for j in range(nk):
            d = int(rng.integers(5, 500))
            kid = f"k{i}_{j}"
            kernels[kid] = KernelEvent(kid, f"kern{rng.integers(0, 20)}", corr, t, t + d, ("main", "fwd"),
                                       {"grid": int(rng.integers(1, 9))} if j == 0 else {})
            corr += 1
            kids.append(kid)
            t += d
        ops.append(OperatorEvent(f"op{i:06d}", f"name{rng.integers(0, 64)}", (), (), tuple(kids), s0, t))
        t += int(rng.integers(0, 30))
    ts = np.arange(10_000 - 50, t + 100, 100)
    w = np.round(rng.uniform(50, 700, size=ts.size), 6)
    w[::7] = 75.0
    power = tuple(PowerSample(int(a), float(b)) for a, b in zip(ts, w))
    return Trace(TraceHeader(1, "A:synthetic", "ingest", seed), {}, tuple(ops), kernels, power, (), None,
                 {"idle_watts": 75.0})


def _same(a: TraceColumns, b: TraceColumns):
    for n in ("ts", "watts", "op_start", "op_end", "k_start", "k_end", "k_op"):
        np.testing.assert_array_equal(a.host(n), b.host(n), err_msg=n)
    assert a.trace_end == b.trace_end
    assert list(a.op_ids) == list(b.op_ids)
    assert list(a.k_ids) == list(b.k_ids)
    assert list(a.op_names) == list(b.op_names)
    assert list(a.k_names) == list(b.k_names)


def test_canonical_scale_trace_parses_on_device(tmp_path):
    tr = _synthetic_trace()
    path = tmp_path / "t.jsonl"
    path.write_text("\n".join(trace_to_lines(tr)) + "\n")
    got = load_columns(path)
    assert got.loaded_by == "gpu"
    _same(got, TraceColumns.from_trace(load_trace(str(path))))
    assert got.header == tr.header and got.config == {"idle_watts": 75.0}
    _same_ranks(got, [o.op_id for o in tr.operators])


def test_no_trailing_newline_and_blank_lines(tmp_path):
    lines = trace_to_lines(_synthetic_trace(200, seed=3))
    path = tmp_path / "t.jsonl"
    path.write_text("\n".join(lines[:5] + ["", "   "] + lines[5:]))
    got = load_columns(path)
    assert got.loaded_by == "gpu"
    _same(got, TraceColumns.from_trace(load_trace(str(path))))


@pytest.mark.parametrize("name", ["tf32_misconfig", "join_redundant"])
def test_reference_traces_with_tensors_parse_on_device(name):
    """Golden reference traces carry tensor snapshots (and a program model):
    power / op / kernel records still parse on the device, only the other
    records are decoded on the host, and the operator-tensor rules hold."""
    for side in ("trace_a", "trace_b"):
        path = GOLDEN / "traces" / name / f"{side}.jsonl"
        got = load_columns(path)
        assert got.loaded_by == "gpu"
        ref = load_trace(str(path))
        _same(got, TraceColumns.from_trace(ref))
        assert got.tensors == ref.tensors and got.progmodel == ref.progmodel
        assert tuple(got.blocktraces) == tuple(ref.blocktraces)
        assert got.op_tensors == [(o.input_tensor_ids, o.output_tensor_ids) for o in ref.operators]
        _same_ranks(got, [o.op_id for o in ref.operators])


def _same_ranks(cols, ids):
    want = np.empty(len(ids), dtype=np.int64)
    want[np.array(sorted(range(len(ids)), key=lambda i: ids[i]), dtype=np.int64)] = np.arange(len(ids))
    np.testing.assert_array_equal(cols.device("op_rank").cpu().numpy(), want)


def test_op_id_ranks_at_ingest(tmp_path):
    """Lexicographic op-id ranks (the report's nodes_a tie-break) on the
    device: ids of different lengths, shared prefixes, multi-word ids."""
    tr = _synthetic_trace(500, seed=9)
    rng = np.random.default_rng(9)
    names = [f"{'x' * int(rng.integers(0, 20))}{rng.integers(0, 10**6)}" + ("_long_suffix" * int(rng.integers(0, 3)))
             for _ in tr.operators]
    names = [f"{n}#{i}" for i, n in enumerate(names)]  # unique
    ops = tuple(OperatorEvent(n, o.op_name, (), (), o.kernel_ids, o.start, o.end) for n, o in zip(names, tr.operators))
    tr = Trace(tr.header, {}, ops, tr.kernels, tr.power, (), None, tr.config)
    path = tmp_path / "t.jsonl"
    path.write_text("\n".join(trace_to_lines(tr)) + "\n")
    got = load_columns(path)
    assert got.loaded_by == "gpu"
    ids = [o.op_id for o in load_trace(str(path)).operators]
    _same_ranks(got, ids)


def _tensor_mutations():
    return {
        "missing_tensor": lambda L: [x for i, x in enumerate(L)
                                     if i != [j for j, y in enumerate(L) if '"type":"tensor"' in y][0]],
        "two_producers": lambda L: _two_producers(L),
    }


def _two_producers(L):
    ops = [i for i, x in enumerate(L) if '"type":"op"' in x]
    L = list(L)
    a, b = json.loads(L[ops[0]]), json.loads(L[ops[1]])
    b["output_tensor_ids"] = list(a["output_tensor_ids"])
    L[ops[1]] = json.dumps(b, separators=(",", ":"))
    return L


@pytest.mark.parametrize("mut", list(_tensor_mutations()))
def test_tensor_rule_violations_raise_the_reference_error(tmp_path, mut):
    src = (GOLDEN / "traces" / "join_redundant" / "trace_a.jsonl").read_text().splitlines()
    lines = _tensor_mutations()[mut](src)
    path = tmp_path / "t.jsonl"
    path.write_text("\n".join(lines) + "\n")
    with pytest.raises(Exception) as want:
        load_trace(str(path))
    with pytest.raises(type(want.value)) as got:
        load_columns(path)
    assert str(got.value) == str(want.value)


def _mutations():
    return {
        "dup_op": lambda L: L + [L[[i for i, x in enumerate(L) if '"type":"op"' in x][0]]],
        "power_order": lambda L: _swap_power(L),
        "neg_watts": lambda L: [x.replace('"watts":75.0', '"watts":-1.0', 1) if '"type":"power"' in x else x
                                for x in L],
        "kernel_outside": lambda L: [x.replace('"end":', '"end":9', 1) if '"type":"kernel"' in x else x for x in L],
        "missing_kernel": lambda L: [x.replace('"kernel_ids":["', '"kernel_ids":["zz', 1) if '"type":"op"' in x else x
                                     for x in L],
        "bad_json": lambda L: L[:3] + ["{not json"] + L[3:],
        "crlf": lambda L: [x + "\r" for x in L],
        "dup_corr": lambda L: _dup_corr(L),
        "big_number": lambda L: [x.replace('"watts":75.0', '"watts":75.00000000000000001', 1) for x in L],
    }


def _swap_power(L):
    idx = [i for i, x in enumerate(L) if '"type":"power"' in x]
    L = list(L)
    L[idx[3]], L[idx[4]] = L[idx[4]], L[idx[3]]
    return L


def _dup_corr(L):
    ks = [i for i, x in enumerate(L) if '"type":"kernel"' in x]
    L = list(L)
    rec = json.loads(L[ks[1]])
    rec["correlation_id"] = json.loads(L[ks[0]])["correlation_id"]
    L[ks[1]] = json.dumps(rec, separators=(",", ":"))
    return L


@pytest.mark.parametrize("mut", list(_mutations()))
def test_broken_files_raise_the_reference_error(tmp_path, mut):
    lines = _mutations()[mut](trace_to_lines(_synthetic_trace(300, seed=5)))
    path = tmp_path / "t.jsonl"
    path.write_bytes(("\n".join(lines) + "\n").encode())
    try:
        want = TraceColumns.from_trace(load_trace(str(path)))
        err = None
    except Exception as exc:  # noqa: BLE001
        want, err = None, exc
    if err is None:
        _same(load_columns(path), want)  # still valid (e.g. a number Python reads fine)
    else:
        with pytest.raises(type(err)) as got:
            load_columns(path)
        assert str(got.value) == str(err)
