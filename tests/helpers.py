"""Shared test helpers (oracle comparison)."""
import numpy as np


def tube_arrays(tube):
    lo = np.stack([e.box.lower for e in tube.entries])
    hi = np.stack([e.box.upper for e in tube.entries])
    return tube.times(), lo, hi


def assert_bitexact(tube, ref):
    t, lo, hi = tube_arrays(tube)
    assert np.array_equal(t, ref.times), (t, ref.times)
    # == semantics: +0 and -0 compare equal (SURVEY.md 8d tolerance contract)
    bad_lo = np.argwhere(lo != ref.lower)
    bad_hi = np.argwhere(hi != ref.upper)
    assert bad_lo.size == 0, f"lower differs at {bad_lo[:5].tolist()}: " \
        f"{lo[tuple(bad_lo[0])]!r} vs {ref.lower[tuple(bad_lo[0])]!r}"
    assert bad_hi.size == 0, f"upper differs at {bad_hi[:5].tolist()}: " \
        f"{hi[tuple(bad_hi[0])]!r} vs {ref.upper[tuple(bad_hi[0])]!r}"


def assert_within(tube, ref, rel=1e-12, atol=0.0):
    """Fast-mode contract: |gpu - ref| <= rel*|ref| + atol per
    bound.  The two-sided bound is also north_star's "never tighter than the
    reference beyond the tolerance": a fast-mode box may be tighter by at most
    rel*|ref| + atol, never by more."""
    t, lo, hi = tube_arrays(tube)
    assert np.array_equal(t, ref.times)
    tol_lo = rel * np.abs(ref.lower) + atol
    tol_hi = rel * np.abs(ref.upper) + atol
    assert np.all(np.abs(lo - ref.lower) <= tol_lo), float(np.max(np.abs(lo - ref.lower) - tol_lo))
    assert np.all(np.abs(hi - ref.upper) <= tol_hi), float(np.max(np.abs(hi - ref.upper) - tol_hi))
