"""Layout-blind tensor equivalence -- drop-in for ``diffwatt.tensor_equiv``.

The reference's criterion (tensor_equiv.py:71-294): two tensors are
equivalent when their element counts match, their Frobenius norms agree, and
the multiset of singular-value spectra of all non-trivial unfoldings of one
embeds injectively into the other's with every matched pair within epsilon
(relative L2 distance); the score is the bottleneck distance of the best
embedding.

The singular values come from the device: ``invariant_sets`` ships every
unfolding of every tensor of a batch to ``dw_unfold_spectra``
(csrc/tensor.cu: one CTA per unfolding, one-sided Jacobi with the reference's
round-robin rotation order, tolerance and sweep cap).  The embedding test
(distance matrix + Kuhn matching + bottleneck search) runs per pair on the
device too (``SpectraBatch.embed`` -> ``dw_spectra_embed``, sets of up to 14
spectra, i.e. order <= 4) with the reference's sequential distance arithmetic;
larger sets use the host restatement below.  Floating point: spectra agree
with the reference's numpy Jacobi to rounding (tests/test_gpu_tensor.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np
import torch

from . import _native

SPECTRUM_FLOOR = 1e-12
DEFAULT_EPSILON = 1e-3
ORDER_CAP = 8
_NORM_FLOOR = 1e-30


@dataclass(frozen=True)
class Spectrum:
    """Singular values sorted descending, trimmed below the floor
    (tensor_equiv.py:30-47)."""

    singulars: tuple

    @classmethod
    def from_values(cls, values: Iterable[float]) -> "Spectrum":
        vals = sorted((float(v) for v in values), reverse=True)
        while vals and vals[-1] < SPECTRUM_FLOOR:
            vals.pop()
        return cls(tuple(vals))

    def norm(self) -> float:
        return math.sqrt(sum(v * v for v in self.singulars))

    def sum_squares(self) -> float:
        return sum(v * v for v in self.singulars)


@dataclass(frozen=True)
class InvariantSet:
    """All unfolding spectra of one tensor (tensor_equiv.py:50-61)."""

    spectra: tuple
    source_order: int

    def frobenius_norm(self) -> float:
        return self.spectra[0].norm() if self.spectra else 0.0


def _arr(t) -> np.ndarray:
    if isinstance(t, np.ndarray):
        return np.asarray(t, dtype=np.float64)
    return np.asarray(t.values, dtype=np.float64).reshape(tuple(t.shape))


def unfold(t, modes: Iterable[int]) -> np.ndarray:
    """Matricization (tensor_equiv.py:71-90): ``modes`` (ascending) index the
    rows, the complement the columns.  Host helper; the device gathers the
    same entries itself."""
    arr = _arr(t)
    r = arr.ndim
    group = sorted(set(int(m) for m in modes))
    if not group:
        raise ValueError("mode subset must be non-empty")
    if any(m < 0 or m >= r for m in group):
        raise ValueError(f"mode out of range for order-{r} tensor")
    if len(group) == r:
        raise ValueError("mode subset must be a proper subset of the modes")
    comp = [m for m in range(r) if m not in group]
    rows = int(np.prod([arr.shape[m] for m in group]))
    return arr.transpose(group + comp).reshape(rows, -1)


# ------------------------------------------------------------ device batch


UNFOLD_DTYPE = np.dtype([("value_off", "<i8"), ("out_off", "<i8"), ("scratch_off", "<i8"), ("order", "<i4"),
                         ("mask", "<i4"), ("dims", "<i4", (8,))])  # dw_unfold_t


class SpectraBatch:
    """Device-resident spectra of every unfolding of a batch of tensors
    (one dw_unfold_spectra launch).  Tensor t owns unfoldings
    set_first[t] .. + set_count[t] (masks 1 .. 2^r - 2 in order); unfolding u
    holds u_len[u] values at spec[u_off[u]:]."""

    def __init__(self, values: np.ndarray, shapes: Sequence[tuple], value_off: Sequence[int]):
        L = _native.lib()
        cap = int(L.dw_unfold_smem_doubles())
        T = len(shapes)
        self.set_count = np.zeros(T, dtype=np.int32)
        self.set_first = np.zeros(T, dtype=np.int64)
        recs, first = [], 0
        order = np.fromiter((len(sh) for sh in shapes), dtype=np.int64, count=T)
        value_off = np.asarray(value_off, dtype=np.int64)
        for r in range(2, ORDER_CAP + 1):
            ts = np.nonzero(order == r)[0]
            if ts.size == 0:
                continue
            D = np.array([shapes[t] for t in ts], dtype=np.int64).reshape(ts.size, r)
            masks = np.arange(1, (1 << r) - 1, dtype=np.int64)
            bits = (masks[:, None] >> np.arange(r)[None, :]) & 1
            rows = np.where(bits[None, :, :] == 1, D[:, None, :], 1).prod(-1)
            total = D.prod(1)[:, None]
            n = np.minimum(rows, total // rows)
            rec = np.zeros((ts.size, masks.size), dtype=UNFOLD_DTYPE)
            rec["value_off"] = value_off[ts][:, None]
            rec["order"] = r
            rec["mask"] = masks[None, :]
            rec["dims"][:, :, :r] = D[:, None, :]
            self.set_first[ts] = first + np.arange(ts.size) * masks.size
            self.set_count[ts] = masks.size
            first += ts.size * masks.size
            recs.append((rec.reshape(-1), n.reshape(-1), (total + n).reshape(-1)))
        self.n_unfold = first
        dev = _native.device()
        if first == 0:
            self.u_off = np.zeros(0, dtype=np.int64)
            self._host = (np.zeros(0), np.zeros(0, dtype=np.int32))
            return
        rec = np.concatenate([x[0] for x in recs])
        n = np.concatenate([x[1] for x in recs])
        need = np.concatenate([x[2] for x in recs])
        out_off = np.zeros(first, dtype=np.int64)
        np.cumsum(n[:-1], out=out_off[1:])
        rec["out_off"] = out_off
        big = need > cap
        scr = np.where(big, need, 0)
        rec["scratch_off"] = np.cumsum(scr) - scr
        smem = int(need[~big].max()) if (~big).any() else 0
        self.u_off = out_off
        self.d_mats = torch.from_numpy(rec.view(np.uint8)).to(dev)
        self.d_vals = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).to(dev)
        self.d_spec = torch.empty(max(int(n.sum()), 1), dtype=torch.float64, device=dev)
        self.d_len = torch.empty(first, dtype=torch.int32, device=dev)
        d_scr = torch.empty(max(int(scr.sum()), 1), dtype=torch.float64, device=dev)
        p = _native.ptr
        _native.check(L.dw_unfold_spectra(p(self.d_vals), p(self.d_mats), first, smem, p(self.d_spec),
                                          p(self.d_len), p(d_scr), _native.stream_handle()), "dw_unfold_spectra")
        self._host = None

    def host(self):
        if self._host is None:
            self._host = (self.d_spec.cpu().numpy(), self.d_len.cpu().numpy())
        return self._host

    def spectra(self, t: int) -> list:
        spec, lens = self.host()
        f = int(self.set_first[t])
        return [Spectrum(tuple(spec[self.u_off[u]:self.u_off[u] + int(lens[u])].tolist()))
                for u in range(f, f + int(self.set_count[t]))]

    def embed(self, job_a: np.ndarray, job_b: np.ndarray, epsilon: float) -> np.ndarray:
        """Bottleneck scores of tensor pairs (job_a[j], job_b[j]) of this batch
        (+inf: no embedding within epsilon) -- dw_spectra_embed."""
        dev = _native.device()
        n = int(job_a.shape[0])
        out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        if n:
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
            keep = [t(self.u_off), self.d_len, t(self.set_first), t(self.set_count), t(job_a.astype(np.int64)),
                    t(job_b.astype(np.int64))]
            p = _native.ptr
            _native.check(_native.lib().dw_spectra_embed(p(self.d_spec), p(keep[0]), p(keep[1]), p(keep[2]),
                                                         p(keep[3]), n, p(keep[4]), p(keep[5]), float(epsilon),
                                                         p(out), _native.stream_handle()), "dw_spectra_embed")
        return out[:n].cpu().numpy()


EMBED_MAX = 14  # DW_EMBED_MAX_SPECTRA: sets up to order 4 embed on the device


def invariant_sets(tensors: Sequence) -> list[InvariantSet]:
    """invariant_set (tensor_equiv.py:162-180) of many tensors at once: every
    unfolding of every tensor in one device launch."""
    arrs = [_arr(t) for t in tensors]
    for a in arrs:
        if a.ndim > ORDER_CAP:
            raise ValueError(f"tensor order {a.ndim} exceeds the cap of {ORDER_CAP}")
    sizes = np.fromiter((a.size for a in arrs), dtype=np.int64, count=len(arrs))
    offs = np.cumsum(sizes) - sizes
    vals = np.concatenate([a.ravel() for a in arrs]) if arrs else np.zeros(0)
    sb = SpectraBatch(vals, [a.shape for a in arrs], offs)
    out = []
    for i, a in enumerate(arrs):
        if a.ndim == 1:
            out.append(InvariantSet((Spectrum.from_values([math.sqrt(float(a @ a))]),), 1))
        elif a.ndim == 0:
            out.append(InvariantSet((), 0))
        else:
            out.append(InvariantSet(tuple(sb.spectra(i)), a.ndim))
    return out


def invariant_set(t) -> InvariantSet:
    return invariant_sets([t])[0]


def singular_values(mat) -> Spectrum:
    """Drop-in for tensor_equiv.singular_values (tensor_equiv.py:113-159)."""
    a = np.asarray(mat, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix has non-finite entries")
    m, n = a.shape
    if min(m, n) == 1:
        v = a.ravel()
        return Spectrum.from_values([math.sqrt(float(v @ v))])
    return SpectraBatch(a.ravel(), [(m, n)], [0]).spectra(0)[0]


# ------------------------------------------------------------- embedding


def spectrum_distance(a: Spectrum, b: Spectrum) -> float:
    """Relative L2 distance, shorter spectrum zero-padded (tensor_equiv.py:183-194)."""
    n = max(len(a.singulars), len(b.singulars))
    if n == 0:
        return 0.0
    diff = 0.0
    for i in range(n):
        va = a.singulars[i] if i < len(a.singulars) else 0.0
        vb = b.singulars[i] if i < len(b.singulars) else 0.0
        diff += (va - vb) ** 2
    return math.sqrt(diff) / max(min(a.norm(), b.norm()), _NORM_FLOOR)


def _distances(small: Sequence[Spectrum], large: Sequence[Spectrum]) -> np.ndarray:
    """The reference's distance matrix (tensor_equiv.py:225-226): every entry
    through spectrum_distance, i.e. the same sequential arithmetic and the same
    norms, so a score at the epsilon / 1% boundary decides as it does there."""
    return np.array([[spectrum_distance(s, l) for l in large] for s in small], dtype=np.float64).reshape(
        len(small), len(large))


def _matching_ok(dist: np.ndarray, limit: float) -> bool:
    """Kuhn augmenting paths: every row takes a distinct column within limit."""
    n_rows, n_cols = dist.shape
    adj = [np.nonzero(dist[i] <= limit)[0].tolist() for i in range(n_rows)]
    owner = [-1] * n_cols

    def augment(i, seen):
        for j in adj[i]:
            if not seen[j]:
                seen[j] = True
                if owner[j] < 0 or augment(owner[j], seen):
                    owner[j] = i
                    return True
        return False

    return all(augment(i, [False] * n_cols) for i in range(n_rows))


def embed_injectively(small: Sequence[Spectrum], large: Sequence[Spectrum], epsilon: float) -> Optional[float]:
    """Bottleneck injective embedding (tensor_equiv.py:219-242): the smallest
    achievable max matched distance if within epsilon, else None."""
    if not small:
        return 0.0
    dist = _distances(small, large)
    levels = np.unique(dist[dist <= epsilon])
    if levels.size == 0 or not _matching_ok(dist, float(levels[-1])):
        return None
    lo, hi = 0, levels.size - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if _matching_ok(dist, float(levels[mid])):
            hi = mid
        else:
            lo = mid + 1
    return float(levels[lo])


def equivalent_from(norm_a: float, norm_b: float, ndim_a: int, ndim_b: int, set_a: Optional[InvariantSet],
                    set_b: Optional[InvariantSet], epsilon: float) -> tuple[bool, float]:
    """tensors_equivalent's decision once counts are known equal and norms and
    invariant sets are computed (tensor_equiv.py:264-294)."""
    nd = abs(norm_a - norm_b) / max(min(norm_a, norm_b), _NORM_FLOOR)
    if nd > epsilon:
        return False, math.inf
    if ndim_a == 1 or ndim_b == 1:
        return nd <= epsilon, nd
    small, large = set_a.spectra, set_b.spectra
    if len(small) > len(large):
        small, large = large, small
    worst = embed_injectively(small, large, epsilon)
    return (False, math.inf) if worst is None else (True, worst)


def tensors_equivalent(a, b, epsilon: float = DEFAULT_EPSILON, set_a: Optional[InvariantSet] = None,
                       set_b: Optional[InvariantSet] = None) -> tuple[bool, float]:
    """Drop-in for tensor_equiv.tensors_equivalent (tensor_equiv.py:245-294)."""
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    xa, xb = _arr(a), _arr(b)
    if xa.size != xb.size:
        return False, math.inf
    # the reference's Frobenius norms, same numpy reduction (tensor_equiv.py:275-276)
    na = float(np.sqrt(np.einsum("i,i->", xa.ravel(), xa.ravel())))
    nb = float(np.sqrt(np.einsum("i,i->", xb.ravel(), xb.ravel())))
    nd = abs(na - nb) / max(min(na, nb), _NORM_FLOOR)
    if nd > epsilon:
        return False, math.inf
    if xa.ndim == 1 or xb.ndim == 1:
        return nd <= epsilon, nd
    need = [x for x, s in ((xa, set_a), (xb, set_b)) if s is None]
    got = iter(invariant_sets(need)) if need else iter(())
    set_a = set_a if set_a is not None else next(got)
    set_b = set_b if set_b is not None else next(got)
    return equivalent_from(na, nb, xa.ndim, xb.ndim, set_a, set_b, epsilon)


def boundary_rel_diff(boundary_right, trace_a, trace_b, limit: float = 0.01) -> float:
    """detect._boundary_rel_diff (detect.py:55-69): worst boundary-tensor diff."""
    from .trace_model import elementwise_rel_diff

    worst = 0.0
    for ta, tb in boundary_right:
        sa, sb = trace_a.snapshot(ta), trace_b.snapshot(tb)
        if tuple(sa.shape) == tuple(sb.shape):
            d = elementwise_rel_diff(sa, sb)
            if d > limit:
                d = min(d, tensors_equivalent(sa, sb, 1.0)[1])
        else:
            d = tensors_equivalent(sa, sb, 1.0)[1]
        worst = max(worst, d)
    return worst
