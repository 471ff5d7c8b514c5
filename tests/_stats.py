"""Aggregate statistical acceptance rule for Monte Carlo estimates.

DESIGN.md reading R14: with r = (est - exact)/SE and
SE from G independent chain groups (r ~ t_{G-1}), require
  (1) mean(r^2) inside a band around E[t^2] = (G-1)/(G-3), widened for the
      number of elements (elements of one estimate are correlated);
  (2) max|r| below the two-sided t_{G-1} Bonferroni quantile at 0.001/count
      (a union bound: valid however the elements' errors are correlated; 0.1%
      per check keeps the rate of a false failure across the suite's ~20
      statistical checks near 2% whenever a realization changes);
  (3) #(|r| > 4) <= 3 * expected + 10.
Complex values contribute their real and imaginary parts as separate elements.
"""
import numpy as np
from scipy import stats


def _flat(est, exact, se):
    est = np.asarray(est).ravel()
    exact = np.asarray(exact).ravel()
    se = np.asarray(se).ravel()
    if np.iscomplexobj(est) or np.iscomplexobj(exact) or np.iscomplexobj(se):
        est = est.astype(np.complex128)
        exact = exact.astype(np.complex128)
        se = se.astype(np.complex128)
        e = np.concatenate([est.real, est.imag])
        x = np.concatenate([exact.real, exact.imag])
        s = np.concatenate([se.real, se.imag])
    else:
        e, x, s = est, exact, se
    # elements that are identically zero in every sample (e.g. Im of a hermitian
    # diagonal) carry only rounding noise: drop them
    keep = s > 1e-9 * (np.max(s) if s.size else 0.0)
    return e[keep], x[keep], s[keep]


def zscores(est, exact, se):
    e, x, s = _flat(est, exact, se)
    return (e - x) / s


def check(est, exact, se, G, what="estimate"):
    r = zscores(est, exact, se)
    count = r.size
    assert count > 0, f"{what}: no element with positive SE"
    e_t2 = (G - 1) / (G - 3) if G > 3 else 3.0
    m2 = float(np.mean(r * r))
    width = 6.0 * np.sqrt(2.0 / count) + 0.25
    assert m2 < e_t2 * (1.0 + width), f"{what}: mean r^2 {m2:.3f} too large (E {e_t2:.3f}, n {count})"
    if count >= 50:
        assert m2 > e_t2 * max(0.05, 1.0 - width), f"{what}: mean r^2 {m2:.3f} too small (SE overstated?)"
    thr = stats.t.ppf(1.0 - 0.0005 / count, G - 1)
    mx = float(np.max(np.abs(r)))
    assert mx < thr, f"{what}: max|r| {mx:.2f} >= Bonferroni {thr:.2f} (n {count}, G {G})"
    p4 = 2 * stats.t.sf(4.0, G - 1)
    n4 = int(np.sum(np.abs(r) > 4))
    assert n4 <= 3 * p4 * count + 10, f"{what}: {n4} elements with |r|>4"
    return dict(mean_r2=m2, max_r=mx, count=count)
