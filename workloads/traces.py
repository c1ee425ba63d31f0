"""Seeded synthetic arrival traces (the workload W).

* Gamma renewal process (reading C17): i.i.d. Gamma(shape=1/CV^2,
  scale=CV^2/rate) gaps -- "a Gamma Process parameterized by rate and
  coefficient of variance (CV)"; CV=1 is the Poisson process of the
  motivating example.
* Power-law per-model split with exponent e: model i gets weight i^-e
  ("power law distribution with an exponent of 0.5").
* MAF1/MAF2-*shaped* windowed rate modulation: the real Azure
  traces are unavailable offline, so per-(model, window) rate factors are
  drawn from a seeded distribution and normalised to mean 1 per model.

All times are float64 seconds until a single round-half-even conversion to
int64 ns (reading C19).  Merging sorts by (arrival_ns, model, per-model seq).
"""

from __future__ import annotations

import numpy as np

from .problem import Trace


def gamma_gaps(rng: np.random.Generator, rate: float, cv: float, n: int) -> np.ndarray:
    shape = 1.0 / (cv * cv)
    scale = cv * cv / rate
    return rng.gamma(shape, scale, size=n)


def gamma_process(rng, rate: float, cv: float, duration: float) -> np.ndarray:
    """Arrival times in [0, duration) of a Gamma renewal process started at 0."""
    if rate <= 0 or duration <= 0:
        return np.zeros(0)
    out = []
    t0 = 0.0
    chunk = int(rate * duration * 1.1) + 64
    while True:
        t = t0 + np.cumsum(gamma_gaps(rng, rate, cv, chunk))
        out.append(t[t < duration])
        if t[-1] >= duration:
            break
        t0 = float(t[-1])
    return np.concatenate(out)


def modulated_gamma_process(rng, rate: float, cv: float, duration: float,
                            window: float, factors: np.ndarray) -> np.ndarray:
    """Gamma renewal process whose rate is rate*factors[w] in window w.

    A unit-rate renewal process in operational time u is mapped through the
    inverse cumulative intensity Lambda^-1 (piecewise linear), so inter-arrival
    CV is preserved within each window and counts follow the window rates."""
    nwin = len(factors)
    edges = np.arange(nwin + 1, dtype=np.float64) * window
    edges[-1] = max(edges[-1], duration)
    lam = rate * np.asarray(factors, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(lam * np.diff(edges))])
    total = float(np.interp(duration, edges, cum))
    u = gamma_process(rng, 1.0, cv, total)
    w = np.clip(np.searchsorted(cum, u, side="right") - 1, 0, nwin - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = edges[w] + np.where(lam[w] > 0, (u - cum[w]) / lam[w], 0.0)
    t = t[t < duration]
    return np.sort(t)


def power_law_weights(num_models: int, exponent: float, rng=None) -> np.ndarray:
    """weights[m] proportional to rank(m)^-exponent, normalised to sum 1; the
    rank permutation is seeded when rng is given."""
    w = np.arange(1, num_models + 1, dtype=np.float64) ** (-float(exponent))
    w /= w.sum()
    if rng is not None:
        w = w[rng.permutation(num_models)]
    return w


def merge(per_model_times, meta=None) -> Trace:
    """Merge per-model float-second arrivals into one sorted int64-ns trace,
    sorted by (arrival_ns, model, per-model sequence) (reading C6)."""
    arrs, mods, seqs = [], [], []
    for m, t in enumerate(per_model_times):
        t = np.asarray(t, dtype=np.float64)
        arrs.append(np.rint(t * 1e9).astype(np.int64))
        mods.append(np.full(len(t), m, dtype=np.int32))
        seqs.append(np.arange(len(t), dtype=np.int64))
    if not arrs:
        return Trace(np.zeros(0, np.int64), np.zeros(0, np.int32), meta or {})
    a = np.concatenate(arrs)
    mo = np.concatenate(mods)
    sq = np.concatenate(seqs)
    order = np.lexsort((sq, mo, a))
    return Trace(np.ascontiguousarray(a[order]), np.ascontiguousarray(mo[order]), meta or {})


def independent_gamma(seed: int, rates, cv: float, duration: float) -> Trace:
    """Independent per-model Gamma processes."""
    rng = np.random.default_rng(seed)
    times = [gamma_process(rng, r, cv, duration) for r in rates]
    return merge(times, dict(kind="independent_gamma", seed=seed, rates=list(map(float, rates)),
                             cv=cv, duration=duration))


def split_gamma(seed: int, total_rate: float, cv: float, duration: float, weights) -> Trace:
    """One Gamma process of the total rate, each request assigned a model with
    probability weights[m] (§5.3: "generated via a Gamma Process ... We
    then split the requests to each model following a power law")."""
    rng = np.random.default_rng(seed)
    t = gamma_process(rng, total_rate, cv, duration)
    w = np.asarray(weights, dtype=np.float64)
    m = rng.choice(len(w), size=len(t), p=w / w.sum())
    times = [t[m == i] for i in range(len(w))]
    return merge(times, dict(kind="split_gamma", seed=seed, total_rate=total_rate, cv=cv,
                             duration=duration))


def maf1_shaped(seed: int, num_models: int, total_rate: float, duration: float,
                exponent: float = 0.5, window: float = 60.0, cv: float = 1.0) -> Trace:
    """MAF1-shaped: "steady and dense incoming requests with gradually changing
    rates".  Power-law base rates over a seeded ranking; 60-s windows
    (P:105 footnote) with factor 1 + 0.5 sin(2 pi t / 86400 + phi_m),
    normalised to mean 1 per model over the trace."""
    rng = np.random.default_rng(seed)
    w = power_law_weights(num_models, exponent, rng)
    nwin = int(np.ceil(duration / window))
    centers = (np.arange(nwin) + 0.5) * window
    times = []
    for m in range(num_models):
        phi = rng.uniform(0, 2 * np.pi)
        f = 1.0 + 0.5 * np.sin(2 * np.pi * centers / 86400.0 + phi)
        f = f / f.mean()
        times.append(modulated_gamma_process(rng, total_rate * w[m], cv, duration, window, f))
    return merge(times, dict(kind="maf1_shaped", seed=seed, total_rate=total_rate,
                             duration=duration, exponent=exponent, window=window, cv=cv))


def maf2_shaped(seed: int, num_models: int, total_rate: float, duration: float,
                exponent: float = 1.0, window: float = 5400.0, cv: float = 4.0,
                sigma: float = 1.0, horizon: float | None = None) -> Trace:
    """MAF2-shaped: "very bursty ... distributed across functions in a highly
    skewed way".  Power-law exponent 1 over a seeded ranking, 5.4 ks
    windows (P:105 footnote) with lognormal(sigma) factors normalised to mean 1
    per model over `horizon` (default: the trace itself), CV 4 within windows.
    A trace shorter than the horizon is its opening stretch: with horizon = one
    day a 1-h trace keeps the day's per-model window factors (a 1-h horizon
    has a single window, whose normalised factor is exactly 1 -- no
    modulation at all)."""
    rng = np.random.default_rng(seed)
    w = power_law_weights(num_models, exponent, rng)
    horizon = duration if horizon is None else max(horizon, duration)
    nwin_h = int(np.ceil(horizon / window))
    nwin = int(np.ceil(duration / window))
    times = []
    for m in range(num_models):
        f = rng.lognormal(0.0, sigma, size=nwin_h)
        f = (f / f.mean())[:nwin]
        times.append(modulated_gamma_process(rng, total_rate * w[m], cv, duration, window, f))
    return merge(times, dict(kind="maf2_shaped", seed=seed, total_rate=total_rate,
                             duration=duration, exponent=exponent, window=window, cv=cv,
                             sigma=sigma, horizon=horizon))
