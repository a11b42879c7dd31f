"""Shared parity helpers for the GPU tests (tests only).

Tolerances (SURVEY.md §8a / BASELINE.json north_star):
* spikes: bit-exact except documented threshold ties — an element may differ
  only where |h2_ref| <= (k+1) 2^-24 (sum_i |w_q,i x| + |b_f|) (fp32 carrier);
* membrane-derived per-channel state (mu, s, a, b_f, running stats): the GPU
  reduces in a different (fixed) order than numpy, so 1e-12 relative;
* gradients dx, dW, dgamma, dbeta in fp32: |got - ref| <= 1e-5 * max(|ref|, 1)
  (pure elementwise relative fails on near-zero dx even for an exact fp32
  kernel);
* float64 carrier: 1e-9 on the same scale.
"""

from __future__ import annotations

import numpy as np

from oracle import psn_oracle as O


def assert_close_scaled(got, ref, tol, what):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    err = np.abs(got - ref)
    bound = tol * np.maximum(np.abs(ref), 1.0)
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} outside {tol}*max(|ref|,1); "
                           f"max err {err.max():.3e}")


def assert_rel(got, ref, tol, what):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref)
    bound = tol * np.maximum(np.abs(ref), np.finfo(np.float64).tiny)
    bad = err > bound
    assert not bad.any(), f"{what}: max rel err {np.max(err / np.maximum(np.abs(ref), 1e-300)):.3e}"


def spikes_match_except_ties(got, ref_out, x, w_q, b_f, d, what="spikes"):
    """Return the number of tie flips; assert every mismatch is a tie."""
    got = np.asarray(got, dtype=np.float64)
    ref_out = np.asarray(ref_out, dtype=np.float64)
    mism = got != ref_out
    if not mism.any():
        return 0
    h2 = O.conv_forward(x.astype(np.float64), w_q, bias=b_f, d=d)
    bound = O.threshold_tie_bound(x, w_q, b_f, d)
    non_tie = mism & (np.abs(h2) > bound)
    assert not non_tie.any(), f"{what}: {int(non_tie.sum())} spike flips that are not threshold ties"
    return int(mism.sum())
