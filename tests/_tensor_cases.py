"""tests/golden/tensors.json.gz (tests/golden/make_golden.py --tensors): the
reference's match_tensors on the classify corpus + two larger scenarios, and
reference invariant sets of seeded random tensors."""

import gzip
import json
from functools import lru_cache

import numpy as np

from _classify_cases import cases as classify_cases
from conftest import GOLDEN
from paper_2512_08365_b200.trace_model import parse_trace_lines


@lru_cache(maxsize=1)
def data() -> dict:
    with gzip.open(GOLDEN / "tensors.json.gz", "rt") as fh:
        return json.load(fh)


def names() -> list:
    return sorted(data()["match"])


@lru_cache(maxsize=64)
def traces(name: str):
    c = data()["traces"].get(name) or classify_cases()[name]
    return parse_trace_lines(c["a"]), parse_trace_lines(c["b"])


def random_tensors():
    r = data()["random"]
    return [(np.asarray(v, dtype=np.float64).reshape(s), sp)
            for s, v, sp in zip(r["shapes"], r["values"], r["spectra"])]
