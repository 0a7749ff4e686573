"""TEST INFRASTRUCTURE ONLY — Lemma 1 (proof P:862-939) evaluated by quadrature.

Two forms:
  * `printed`   — Lemma 1 exactly as typeset: recycled-job term integrates
                  t from r + a0 (a0 = C r of the TAGGED job), residence to a0, final
                  term (x - a0).
  * `corrected` — the SOAP Theorem 5.5 assembly of the same model with the
                  old job's OWN threshold (reading D-19): an old job I with r_I = y > r
                  becomes recycled at age s(y) = min(y - r, C y) (rank crossing r, or its
                  own a0_I = C y, whichever first) and then runs to completion, so
                    M1(r) = int_{y>r} int_{x>s(y)} (x - s(y))^2 g(x,y) dx dy,
                  residence = int_0^{min(x, a0)} da / (1 - rho'_{(r-a)+}) + (x - a0)^+.
Both use rho'_r = lam int_0^r int x g(x,y) dx dy and M0(r) = int_0^r int x^2 g dx dy.
C = 0 literally makes every rank -inf: all jobs tie and FCFS applies, so E[T]
is Pollaczek-Khinchine; C -> 0+ (zero_plus) is non-preemptive SPJF (reading D-13).

Service f(x) = e^{-x} (App. D).  Predictors (App. D):
  'perfect'      g(x,y) = e^{-x} delta(y - x)
  'exponential'  g(x,y) = e^{-x} (1/x) e^{-y/x}   (typo e^{(-x-y)/x} fixed)
Integrals over the exponential predictor substitute y = x u (u ~ Exp(1)), which removes
the 1/x singularity.  Composite Gauss-Legendre throughout, split at every kink.
"""
from __future__ import annotations

import numpy as np

U_MAX = 45.0            # e^{-45} ~ 3e-20: truncation of the Exp(1) tails
_GL_CACHE = {}


def _gl(npts: int):
    if npts not in _GL_CACHE:
        _GL_CACHE[npts] = np.polynomial.legendre.leggauss(npts)
    return _GL_CACHE[npts]


def _gl_nodes(a, b, npts: int = 48):
    """Nodes/weights on [a, b] (broadcast over arrays a, b): shapes a.shape + (npts,)."""
    t, w = _gl(npts)
    a = np.asarray(a, dtype=np.float64)[..., None]
    b = np.asarray(b, dtype=np.float64)[..., None]
    half = 0.5 * (b - a)
    return a + half * (t + 1.0), half * w


def _composite(a: float, b: float, panels: int, npts: int = 24):
    edges = np.linspace(a, b, panels + 1)
    x, w = _gl_nodes(edges[:-1], edges[1:], npts)
    return x.ravel(), w.ravel()


# ----------------------------------------------------------------------------- pieces
class _Model:
    def __init__(self, lam: float, predictor: str):
        if predictor not in ("perfect", "exponential"):
            raise ValueError(predictor)
        self.lam, self.pred = float(lam), predictor
        # outer x-grid for the exponential predictor's inner integrals over x
        self.xg, self.xw = _composite(0.0, U_MAX, 150, 12)

    # rho'_r and M0(r) (vectorised over r)
    def rho(self, r):
        r = np.asarray(r, dtype=np.float64)
        if self.pred == "perfect":
            x, w = _gl_nodes(np.zeros_like(r), np.minimum(r, U_MAX), 64)
            return self.lam * np.sum(w * x * np.exp(-x), axis=-1)
        x, w = self.xg, self.xw                      # P(Y < r | x) = 1 - e^{-r/x}
        pr = -np.expm1(-r[..., None] / x)
        return self.lam * np.sum(w * x * np.exp(-x) * pr, axis=-1)

    def m0(self, r):
        r = np.asarray(r, dtype=np.float64)
        if self.pred == "perfect":
            x, w = _gl_nodes(np.zeros_like(r), np.minimum(r, U_MAX), 64)
            return np.sum(w * x * x * np.exp(-x), axis=-1)
        x, w = self.xg, self.xw
        pr = -np.expm1(-r[..., None] / x)
        return np.sum(w * x * x * np.exp(-x) * pr, axis=-1)

    def m1_corrected(self, r, C: float):
        """int_{y>r} int_{x > s(y)} (x - s(y))^2 g(x,y), s(y) = min(y - r, C y)."""
        r = np.atleast_1d(np.asarray(r, dtype=np.float64))
        if self.pred == "perfect":
            # x = y; x - s(y) = max(r, (1-C) y) > 0.  Kink at y = r/(1-C) when C < 1.
            out = np.zeros_like(r)
            for i, ri in enumerate(r):
                brk = [ri, U_MAX + ri]
                if C < 1.0 and ri / (1.0 - C) < brk[-1]:
                    brk.insert(1, ri / (1.0 - C))
                tot = 0.0
                for a, b in zip(brk[:-1], brk[1:]):
                    y, w = _composite(a, b, 8, 24)
                    v = np.maximum(ri, (1.0 - C) * y)
                    tot += np.sum(w * v * v * np.exp(-y))
                out[i] = tot
            return out
        out = np.zeros_like(r)
        x = self.xg[:, None]
        xw = self.xw[:, None]
        for i, ri in enumerate(r):
            # u from r/x to r/x + U_MAX; kinks: s switches at u = r/(x(1-C));
            # (x - s)^+ vanishes past u where s = x: u = (x+r)/x (rank branch) or 1/C.
            lo = ri / x
            hi = lo + U_MAX
            cands = [lo, hi, np.clip((x + ri) / x, lo, hi)]
            if C > 0:
                cands.append(np.clip(np.full_like(x, 1.0 / C), lo, hi))
            if C < 1.0:
                cands.append(np.clip(ri / (x * (1.0 - C)), lo, hi))
            bk = np.sort(np.concatenate(cands, axis=1), axis=1)
            tot = 0.0
            for s in range(bk.shape[1] - 1):
                u, w = _gl_nodes(bk[:, s], bk[:, s + 1], 24)
                y = x * u
                sv = np.minimum(y - ri, C * y)
                v = np.maximum(x - sv, 0.0)
                tot += np.sum(xw * np.exp(-x) * np.sum(w * np.exp(-u) * v * v, axis=1, keepdims=True))
            out[i] = tot
        return out

    def m1_printed(self, r, C: float):
        """int_{t = r + a0}^inf int_{x > t - r} g(x,t) (x - (t - r))^2, a0 = C r."""
        r = np.atleast_1d(np.asarray(r, dtype=np.float64))
        a0 = C * r
        if self.pred == "perfect":      # x = t: (x - (t - r))^2 = r^2, mass e^{-(r + a0)}
            return r * r * np.exp(-(r + a0))
        out = np.zeros_like(r)
        x = self.xg[:, None]
        xw = self.xw[:, None]
        for i, ri in enumerate(r):
            lo = (ri + a0[i]) / x            # t = x u >= r + a0
            hi = (x + ri) / x                # x > t - r  <=>  u < (x + r)/x
            hi = np.maximum(hi, lo)
            u, w = _gl_nodes(lo[:, 0], hi[:, 0], 32)
            v = x - (x * u - ri)
            out[i] = np.sum(xw * np.exp(-x) * np.sum(w * np.exp(-u) * v * v, axis=1, keepdims=True))
        return out


def _residence_table(model: _Model, rmax: float, npts: int = 4001):
    """F(r) = int_0^r dv / (1 - rho'_v) on a grid (cumulative composite Simpson)."""
    rg = np.linspace(0.0, rmax, npts)
    f = 1.0 / (1.0 - model.rho(rg))
    F = np.zeros_like(rg)
    h = rg[1] - rg[0]
    F[1:] = np.cumsum(0.5 * h * (f[1:] + f[:-1]))
    # refine trapezoid with one Richardson step on a half grid
    rh = np.linspace(0.0, rmax, 2 * (npts - 1) + 1)
    fh = 1.0 / (1.0 - model.rho(rh))
    Fh = np.zeros_like(rh)
    Fh[1:] = np.cumsum(0.5 * (rh[1] - rh[0]) * (fh[1:] + fh[:-1]))
    return rg, Fh[::2] + (Fh[::2] - F) / 3.0


def mean_response(lam: float, C: float, predictor: str = "perfect", form: str = "corrected",
                  zero_plus: bool = False) -> float:
    """E[T] = int int g(x,y) E[T(x,y)] for Exp(1) service."""
    if C == 0.0 and not zero_plus:           # every rank is -inf: FCFS, P-K (D-13)
        return lam * 2.0 / (2.0 * (1.0 - lam)) + 1.0
    model = _Model(lam, predictor)
    Ceff = 0.0 if zero_plus else float(C)
    # tabulate W(r) = lam (M0 + M1) / (2 (1 - rho'_r)^2) and F(r)
    rg = np.concatenate([np.linspace(0, 4, 161)[:-1], np.linspace(4, 20, 161)[:-1],
                         np.linspace(20, 60, 81)])
    rho = model.rho(rg)
    m0 = model.m0(rg)
    if zero_plus:                             # old jobs with y > r: full size, s = 0
        m1 = model.m1_corrected(rg, 0.0)
    elif form == "corrected":
        m1 = model.m1_corrected(rg, Ceff)
    else:
        m1 = model.m1_printed(rg, Ceff)
    W = lam * (m0 + m1) / (2.0 * (1.0 - rho) ** 2)
    Fr, F = _residence_table(model, 60.0)

    def wait(y):
        return np.interp(y, rg, W)

    def resid(x, y):
        a0 = Ceff * y
        if form == "corrected":
            A = np.minimum(x, a0)
            tail = np.maximum(x - a0, 0.0)
        else:
            A = a0
            tail = x - a0
        Ain = np.minimum(A, y)                 # (r - a)^+ hits 0 after a = r: integrand 1
        return (np.interp(y, Fr, F) - np.interp(y - Ain, Fr, F)) + (A - Ain) + tail

    if predictor == "perfect":
        x, w = _composite(0.0, U_MAX, 180, 24)
        return float(np.sum(w * np.exp(-x) * (wait(x) + resid(x, x))))
    # exponential predictor: y = x u; split u at 1/C (kink of min(x, C y))
    x, xw = _composite(0.0, U_MAX, 180, 16)
    tot = 0.0
    brk = [0.0, U_MAX]
    if Ceff > 0 and 1.0 / Ceff < U_MAX:
        brk = [0.0, 1.0 / Ceff, U_MAX]
    for a, b in zip(brk[:-1], brk[1:]):
        u, uw = _composite(a, b, 60, 16)
        X = x[:, None]
        Y = X * u[None, :]
        val = wait(Y) + resid(X, Y)
        tot += np.sum(xw[:, None] * np.exp(-X) * uw[None, :] * np.exp(-u)[None, :] * val)
    return float(tot)
