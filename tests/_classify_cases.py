"""The reference's classify golden cases (tests/golden/classify.json.gz, made
by tests/golden/make_golden.py --classify): traces as JSONL lines and, per
detect_waste finding, (nodes_a, nodes_b, verdict, side, category,
forced_gap_joules of the wasteful side)."""

import gzip
import json
from functools import lru_cache

from conftest import GOLDEN
from paper_2512_08365_b200.detect import SubgraphPair, WasteFinding
from paper_2512_08365_b200.trace_model import parse_trace_lines


@lru_cache(maxsize=1)
def cases() -> dict:
    with gzip.open(GOLDEN / "classify.json.gz", "rt") as fh:
        return json.load(fh)


@lru_cache(maxsize=64)
def traces(name: str):
    c = cases()[name]
    return parse_trace_lines(c["a"]), parse_trace_lines(c["b"])


def findings(name: str) -> list:
    """Reference-shaped findings carrying the reference's verdict and side
    (category left "unknown" for the classifier under test)."""
    out = []
    for na, nb, verdict, side, _, _ in cases()[name]["findings"]:
        out.append(WasteFinding(pair=SubgraphPair(tuple(na), tuple(nb)), energy_a=0.0, energy_b=0.0,
                                energy_ratio=1.0, latency_a=0, latency_b=0, output_rel_diff=0.0,
                                verdict=verdict, category="unknown", wasteful_side=side,
                                wasted_joules=0.0, informational=False))
    return out
