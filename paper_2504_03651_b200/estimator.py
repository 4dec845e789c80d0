"""Batch execution-time estimator of the paper (§5.2), calibrated on THIS library's
B200 kernels.  Host-side numerics only (numpy least squares); it consumes
timings of hybrid_attention measured by profiles/calibrate.py and never runs on the hot path.

Models (equation numbers as printed in PAPER.md; SPEC.md numbers them 5-7):
  Eq.(6)  Time_prefill = max(alpha*l^2 + beta*l, c)
          chunk [s, e): max(alpha*(e^2 - s^2) + beta*(e - s), c)  (marginal cost)
  Eq.(7)  Time_decode  = gamma*max(L) + delta*mean(L)
  Eq.(8)  Time_batch   = lambda*max(Tp, Td) + (1 - lambda)*min(Tp, Td)
          (a pure batch returns its nonzero component; lambda unconstrained)

The calibration follows S:262-267: (alpha, beta, c) on pure-prefill samples (c by a grid over
floor candidates, alpha/beta by linear least squares on above-floor samples), (gamma, delta) by
linear least squares on pure-decode samples, lambda by 1-D least squares on mixed samples.  All
fits minimise RELATIVE residuals (timing noise is multiplicative), so short batches weigh as
much as long ones.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np


class CalibrationError(ValueError):
    """Insufficient sample diversity for a regime of the model."""


@dataclass
class Params:
    alpha: float
    beta: float
    c: float
    gamma: float
    delta: float
    lam: float
    mu: float = 0.0   # prose form of Eq.(8): max + mu*min ("greater than the maximum ... less than their sum")

    def as_dict(self):
        d = asdict(self)
        d["lambda"] = d.pop("lam")
        return d


def prefill_time(start: float, end: float, p: Params) -> float:
    """Eq.(6) for the chunk [start, end): marginal quadratic + linear cost, floor c."""
    if not (0 <= start < end):
        raise ValueError("prefill_time needs 0 <= start < end")
    return max(p.alpha * (end * end - start * start) + p.beta * (end - start), p.c)


def decode_time(L, p: Params) -> float:
    """Eq.(7): gamma * max(L) + delta * mean(L)."""
    L = np.asarray(L, dtype=np.float64)
    if L.size == 0 or (L < 1).any():
        raise ValueError("decode_time needs a non-empty L with all lengths >= 1")
    return p.gamma * float(L.max()) + p.delta * float(L.mean())


def batch_time(tp: float, td: float, p: Params) -> float:
    """Eq.(8) as written; a pure batch returns its nonzero component."""
    if tp < 0 or td < 0:
        raise ValueError("components must be >= 0")
    if tp == 0 or td == 0:
        return tp + td
    return p.lam * max(tp, td) + (1.0 - p.lam) * min(tp, td)


def batch_time_prose(tp: float, td: float, p: Params) -> float:
    """The reading of Eq.(8) that matches its prose (S:288 open question): the mixed time
    lies between max and sum, T = max(Tp, Td) + mu * min(Tp, Td), mu in [0, 1]."""
    if tp < 0 or td < 0:
        raise ValueError("components must be >= 0")
    return max(tp, td) + p.mu * min(tp, td)


def sample_components(s: dict, p: Params):
    """(Tp, Td) of a profile sample {"prefill_spans": [[s, e], ...], "decode_lens": [...]}:
    prefills are charged one by one ("process prefill requests one by one")."""
    tp = sum(prefill_time(a, b, p) for a, b in s.get("prefill_spans", []))
    L = s.get("decode_lens", [])
    td = decode_time(L, p) if len(L) else 0.0
    return tp, td


def estimate(s: dict, p: Params) -> float:
    tp, td = sample_components(s, p)
    return batch_time(tp, td, p)


def calibrate(samples, floor_grid: int = 64) -> Params:
    """Least-squares calibration.  samples: dicts with prefill_spans, decode_lens,
    time_s.  Raises CalibrationError naming a missing regime."""
    pre = [s for s in samples if s.get("prefill_spans") and not s.get("decode_lens")]
    dec = [s for s in samples if s.get("decode_lens") and not s.get("prefill_spans")]
    mix = [s for s in samples if s.get("decode_lens") and s.get("prefill_spans")]
    if len(pre) < 3:
        raise CalibrationError("need >= 3 pure-prefill samples")
    if len(dec) < 2:
        raise CalibrationError("need >= 2 pure-decode samples")
    if len(mix) < 1:
        raise CalibrationError("need >= 1 mixed sample")

    # (alpha, beta, c): single-span prefill samples; c over a grid of floor candidates, alpha /
    # beta by least squares on the samples above the candidate floor
    q = np.array([sum(b * b - a * a for a, b in s["prefill_spans"]) for s in pre], np.float64)
    lin = np.array([sum(b - a for a, b in s["prefill_spans"]) for s in pre], np.float64)
    t = np.array([s["time_s"] for s in pre], np.float64)
    if np.linalg.matrix_rank(np.stack([q, lin], 1)) < 2:
        raise CalibrationError("pure-prefill samples do not separate the l^2 and l terms")
    cands = np.unique(np.concatenate([[0.0], np.sort(t)[: max(1, len(t) // 2)]]))
    if len(cands) > floor_grid:
        cands = cands[np.linspace(0, len(cands) - 1, floor_grid).astype(int)]
    best = None
    for c in cands:
        above = t > c * (1 + 1e-9)
        if above.sum() < 2 or np.linalg.matrix_rank(np.stack([q[above], lin[above]], 1)) < 2:
            continue
        w = 1.0 / t[above]  # relative (multiplicative-noise) least squares
        (al, be), *_ = np.linalg.lstsq(np.stack([q[above], lin[above]], 1) * w[:, None], t[above] * w,
                                       rcond=None)
        al, be = max(al, 0.0), max(be, 0.0)
        pred = np.maximum(al * q + be * lin, c)
        err = float((((pred - t) / t) ** 2).sum())
        if best is None or err < best[0]:
            best = (err, al, be, float(c))
    if best is None:
        raise CalibrationError("no floor candidate leaves two independent above-floor prefill samples")
    _, alpha, beta, c = best

    # (gamma, delta): pure-decode samples
    mx = np.array([max(s["decode_lens"]) for s in dec], np.float64)
    mn = np.array([np.mean(s["decode_lens"]) for s in dec], np.float64)
    td = np.array([s["time_s"] for s in dec], np.float64)
    A = np.stack([mx, mn], 1)
    if np.linalg.matrix_rank(A) < 2:
        raise CalibrationError("pure-decode samples do not separate max(L) from mean(L)")
    # relative least squares under the SPEC invariant gamma, delta >= 0 (CostModelParams): a
    # two-variable NNLS — the unconstrained optimum if it is feasible, else the better of the
    # two one-coefficient fits on the boundary (KKT for a convex quadratic with two bounds)
    Aw, bw = A / td[:, None], np.ones_like(td)
    (gamma, delta), *_ = np.linalg.lstsq(Aw, bw, rcond=None)
    if gamma < 0 or delta < 0:
        cand = []
        for j in (0, 1):
            col = Aw[:, j]
            x = max(float(col @ bw / (col @ col)), 0.0)
            sol = [0.0, 0.0]
            sol[j] = x
            cand.append((float(((Aw @ np.array(sol)) - bw) @ ((Aw @ np.array(sol)) - bw)), sol))
        gamma, delta = min(cand)[1]

    # lambda: 1-D least squares on mixed samples, T = lam*(max - min) + min
    p0 = Params(alpha, beta, c, float(gamma), float(delta), 0.0)
    comps = [sample_components(s, p0) for s in mix]
    hi = np.array([max(a, b) for a, b in comps])
    lo = np.array([min(a, b) for a, b in comps])
    tm = np.array([s["time_s"] for s in mix], np.float64)
    dd = (hi - lo) / tm
    lam = float((dd * ((tm - lo) / tm)).sum() / (dd * dd).sum()) if (dd * dd).sum() > 0 else 1.0
    # prose form: T = max + mu*min
    lr = lo / tm
    mu = float((lr * ((tm - hi) / tm)).sum() / (lr * lr).sum()) if (lr * lr).sum() > 0 else 0.0
    return Params(float(alpha), float(beta), float(c), float(gamma), float(delta), lam, mu)
