"""paper_2512_08365_b200 -- B200-native hot path of Magneton / diffwatt.

Drop-in for the analysis hot path of the reference package
(/root/reference/pkg/src/diffwatt): trace ingestion into columnar device
buffers, per-operator energy attribution, the cross-system differential diff
and ranked findings.  The compute runs in hand-written sm_100a CUDA kernels
(csrc/, exported through the C ABI in include/dwb200.h); there is no CPU
fallback.
"""

from .trace_model import (  # noqa: F401
    KernelEvent,
    OperatorEvent,
    ParseError,
    PowerSample,
    Trace,
    TraceError,
    TraceHeader,
    TraceReferenceError,
    VersionError,
    load_trace,
    parse_trace_lines,
    save_trace,
    trace_to_lines,
)
from .columns import TraceColumns  # noqa: F401
from .energy import (  # noqa: F401
    EnergyLedger,
    PowerSignal,
    ReplayEstimate,
    SignalError,
    build_ledger,
    ground_truth_signal,
    integrate,
    integrate_many,
    integrate_split,
    mean_power,
    replay_estimate,
    sample_signal,
    sampled_view,
)

from .detect import (  # noqa: F401
    Report,
    SubgraphPair,
    WasteFinding,
    detect_waste,
    report,
)
from .diagnose import (  # noqa: F401
    DiagnoseError,
    classify,
    classify_findings,
    forced_gap_joules,
    idle_baseline_watts,
)
from .join import join_diff, join_report, signature_of  # noqa: F401
from .pipeline import analyze, analyze_corpus  # noqa: F401
from .tensor_equiv import invariant_set, invariant_sets, singular_values, tensors_equivalent  # noqa: F401
from .tensor_match import MatchStats, TensorPair, TensorPairSet, match_tensors  # noqa: F401

__version__ = "0.1.0"
