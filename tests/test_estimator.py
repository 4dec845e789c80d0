"""Pins for the batch-time estimator (Eq.(6)-(8)), host only.

* SPEC examples, each a direct evaluation of the printed formula.
* Calibration round trip: samples generated from known parameters are recovered
  within 1% without noise and within 10% (median over 20 seeds) with 5% multiplicative noise;
  a missing regime raises CalibrationError.
"""
import numpy as np
import pytest

from paper_2504_03651_b200 import estimator as E

P = E.Params(alpha=2e-7, beta=1e-4, c=5e-3, gamma=1e-6, delta=2e-5, lam=0.9)


def test_spec_examples():
    assert E.prefill_time(0, 1000, P) == pytest.approx(0.3, rel=1e-12)
    assert E.prefill_time(0, 8, P) == pytest.approx(5e-3, rel=1e-12)              # S:232 floor
    big = E.Params(2e-7, 1e-4, 1e-6, 0, 0, 0)
    assert E.prefill_time(0, 500, big) + E.prefill_time(500, 1000, big) == pytest.approx(
        E.prefill_time(0, 1000, big), rel=1e-12)
    assert E.decode_time([100, 200, 300], P) == pytest.approx(4.3e-3, rel=1e-12)
    assert E.decode_time([77], P) == pytest.approx((P.gamma + P.delta) * 77, rel=1e-12)
    assert E.decode_time([300, 100, 200], P) == E.decode_time([100, 200, 300], P)
    assert E.batch_time(0.3, 0.0043, P) == pytest.approx(0.27043, rel=1e-12)
    assert E.batch_time(0.3, 0.0, P) == 0.3
    p1 = E.Params(0, 0, 0, 0, 0, 1.0)
    assert E.batch_time(0.3, 0.2, p1) == 0.3
    with pytest.raises(ValueError):
        E.prefill_time(10, 10, P)
    with pytest.raises(ValueError):
        E.decode_time([], P)


def _samples(p, rng, noise=0.0):
    out = []
    for l in [4, 16, 48, 64, 96, 128, 192, 256, 512, 1024, 2048, 4096, 8192]:
        out.append({"prefill_spans": [[0, l]], "decode_lens": []})
    for _ in range(12):  # uniform batches and batches with one long outlier (max != mean)
        n = int(rng.integers(2, 64))
        L = rng.integers(16, 512, n).tolist()
        if rng.random() < 0.5:
            L[0] = int(rng.integers(4096, 32768))
        out.append({"prefill_spans": [], "decode_lens": L})
    for _ in range(8):
        l = int(rng.integers(256, 4096))
        L = rng.integers(16, 4096, int(rng.integers(1, 64))).tolist()
        out.append({"prefill_spans": [[0, l]], "decode_lens": L})
    for s in out:
        s["time_s"] = E.estimate(s, p) * (1 + noise * rng.standard_normal())
    return out


def _rel(a, b):
    return abs(a - b) / abs(b)


def test_calibration_round_trip_noiseless():
    s = _samples(P, np.random.default_rng(0))
    f = E.calibrate(s)
    for k in ("alpha", "beta", "c", "gamma", "delta", "lam"):
        assert _rel(getattr(f, k), getattr(P, k)) < 0.01, k


def test_calibration_noisy_median_within_10pct():
    errs = {k: [] for k in ("alpha", "beta", "c", "gamma", "delta", "lam")}
    for seed in range(20):
        f = E.calibrate(_samples(P, np.random.default_rng(100 + seed), noise=0.05))
        for k in errs:
            errs[k].append(_rel(getattr(f, k), getattr(P, k)))
    for k, v in errs.items():
        assert np.median(v) < 0.10, (k, np.median(v))


def test_calibration_missing_regime():
    s = _samples(P, np.random.default_rng(1))
    with pytest.raises(E.CalibrationError):
        E.calibrate([x for x in s if not x["decode_lens"]])          # all-prefill
    with pytest.raises(E.CalibrationError):
        E.calibrate([x for x in s if not x["prefill_spans"]])        # all-decode


def test_prose_form_round_trip():
    """The prose reading of Eq.(8) (max + mu*min) is recovered from samples made with it."""
    p = E.Params(2e-7, 1e-4, 5e-3, 1e-6, 2e-5, 0.9, mu=0.3)
    rng = np.random.default_rng(5)
    s = _samples(p, rng)
    for x in s:
        if x["prefill_spans"] and x["decode_lens"]:
            tp, td = E.sample_components(x, p)
            x["time_s"] = E.batch_time_prose(tp, td, p)
    f = E.calibrate(s)
    assert _rel(f.mu, 0.3) < 0.01
    assert E.batch_time_prose(0.3, 0.1, p) == pytest.approx(0.33, rel=1e-12)


def test_calibration_params_nonnegative_under_noise():
    """SPEC CostModelParams invariant (gamma, delta >= 0): decode samples whose noise makes the
    unconstrained fit put a negative weight on max(L) still calibrate to non-negative
    coefficients, and decode_time stays monotone in every L."""
    rng = np.random.default_rng(3)
    base = _samples(P, rng)
    dec = []
    for _ in range(8):    # max(L) anti-correlated with time: unconstrained gamma < 0
        n = int(rng.integers(4, 40))
        lens = list(rng.integers(50, 400, n))
        lens[0] = int(rng.integers(400, 4000))
        t = 2e-5 * float(np.mean(lens)) * (1 + 0.05 * rng.standard_normal()) - 1e-7 * lens[0] + 1e-4
        dec.append({"prefill_spans": [], "decode_lens": lens, "time_s": max(t, 1e-6)})
    samples = [s for s in base if not (s["decode_lens"] and not s["prefill_spans"])] + dec
    raw, *_ = np.linalg.lstsq(np.array([[max(s["decode_lens"]), np.mean(s["decode_lens"])] for s in dec])
                              / np.array([s["time_s"] for s in dec])[:, None], np.ones(len(dec)), rcond=None)
    assert min(raw) < 0        # the case the constraint exists for
    fit = E.calibrate(samples)
    assert fit.gamma >= 0 and fit.delta >= 0
    assert E.decode_time([100, 200], fit) <= E.decode_time([100, 300], fit)
