"""Oracle: SVD-based compressors of the Appendix.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  complex128 throughout.

Truncation rule (reading Q7 of SURVEY.md / DESIGN.md): at every truncated
SVD the kept rank is
    r = min{ r >= 1 : || sigma_{r+1:} ||_2 <= delta },
with delta = (gamma / sqrt(#truncations)) * ||T||_F, #truncations = d for
Alg. 1, d-1 for Alg. 3 and 6 for Alg. 2 (reading Q8:
the leaves of Alg. 2 also use gamma/sqrt(6)).  Equality keeps the smaller r.
This makes the reconstruction-error bound ||T - T_hat||_F <= gamma ||T||_F
a theorem (each truncation contributes at most delta^2 to the squared error).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from .tensor import frob, mode_product, unfold


@dataclasses.dataclass
class Truncation:
    rank: int
    sigma: np.ndarray     # all singular values of the unfolding (descending)
    delta: float          # absolute threshold
    margin: float         # min relative distance of the tail norms to delta around the decision


def tail_rank(sigma: np.ndarray, delta: float) -> Truncation:
    """r = min{r >= 1 : ||sigma[r:]||_2 <= delta}  (reading Q7)."""
    s = np.asarray(sigma, dtype=np.float64)
    sq = s * s
    # tails[r] = sqrt(sum_{j >= r} sigma_j^2), r = 0..len(s)
    tails = np.sqrt(np.concatenate([np.cumsum(sq[::-1])[::-1], [0.0]]))
    r = len(s)
    for cand in range(1, len(s) + 1):
        if tails[cand] <= delta:
            r = cand
            break
    if delta > 0:
        m = abs(tails[r] - delta) / delta
        if r > 1:
            m = min(m, abs(tails[r - 1] - delta) / delta)
    else:
        m = math.inf
    return Truncation(r, s, float(delta), float(m))


def svd(a: np.ndarray):
    """Thin SVD (library primitive)."""
    return np.linalg.svd(a, full_matrices=False)


# --------------------------------------------------------------------------- Alg. 1
@dataclasses.dataclass
class TuckerFormat:
    core: np.ndarray               # r1 x .. x rd
    factors: list                  # U^i, n_i x r_i
    truncations: list              # per-mode Truncation

    @property
    def ranks(self):
        return tuple(self.core.shape)


def tucker_svd(t: np.ndarray, gamma: float, n_trunc: int | None = None,
               norm: float | None = None) -> TuckerFormat:
    """Alg. 1 Tucker-SVD (classical HOSVD).

    For i = 1..d: SVD of the mode-i unfolding of T (step 5-6), rank r_i by the
    tail rule with delta = gamma/sqrt(d) ||T||_F (step 7), U^i = leading r_i
    left singular vectors; C = T x_1 U^1* x_2 ... x_d U^d* (step 8, * = conjugate
    transpose; the projection reading of SURVEY.md Q9).
    `n_trunc` overrides sqrt(d) (Alg. 2 uses 6); `norm` overrides ||T||_F.
    """
    d = t.ndim
    n_trunc = d if n_trunc is None else n_trunc
    nrm = frob(t) if norm is None else norm
    delta = gamma / math.sqrt(n_trunc) * nrm
    factors, truncs = [], []
    for i in range(1, d + 1):
        u, s, _ = svd(unfold(t, i))
        tr = tail_rank(s, delta)
        factors.append(u[:, :tr.rank].copy())
        truncs.append(tr)
    core = t
    for i, u in enumerate(factors, start=1):
        core = mode_product(core, u.conj().T, i)
    return TuckerFormat(core, factors, truncs)


# --------------------------------------------------------------------------- Alg. 3
@dataclasses.dataclass
class TTFormat:
    head: np.ndarray          # U^1_TT, n1 x r1
    cores: list               # C^i_TT, r_i x n_{i+1} x r_{i+1}  (d-2 of them)
    tail: np.ndarray          # U^last_TT, n_d x r_{d-1}
    truncations: list

    @property
    def ranks(self):
        return tuple(tr.rank for tr in self.truncations)


def tt_svd(t: np.ndarray, gamma: float) -> TTFormat:
    """Alg. 3 TT-SVD: sequential left-to-right truncated SVDs of
    the running remainder, delta = gamma/sqrt(d-1) ||T||_F.  Core i is the
    truncated U reshaped (r_{i-1}, n_i, r_i) (step 7); the remainder is
    Sigma V* (step 8).  The first core is the head factor U^1 (n1 x r1); the
    last remainder, transposed, is the tail factor (n_d x r_{d-1}) (step 10,
    reading Q11)."""
    d = t.ndim
    n = t.shape
    delta = gamma / math.sqrt(d - 1) * frob(t)
    c = np.reshape(t, (n[0], -1), order="F")
    r_prev = 1
    cores, truncs = [], []
    for i in range(d - 1):
        c = np.reshape(c, (r_prev * n[i], -1), order="F")    # step 5
        u, s, vh = svd(c)                                     # step 6
        tr = tail_rank(s, delta)                              # step 7
        r = tr.rank
        cores.append(np.reshape(u[:, :r], (r_prev, n[i], r), order="F"))
        c = s[:r, None] * vh[:r, :]                           # step 8
        truncs.append(tr)
        r_prev = r
    head = cores[0][0]                                        # (n1, r1)
    tail = c.T.copy()                                         # (n_d, r_{d-1})
    return TTFormat(head, cores[1:], tail, truncs)


# --------------------------------------------------------------------------- Alg. 2
@dataclasses.dataclass
class HTuckerFormat:
    leaves: list              # U^i_HT, n_i x r_i, i = 1..4
    c12: np.ndarray           # r1 x r2 x r12
    c34: np.ndarray           # r3 x r4 x r34
    c1234: np.ndarray         # r12 x r34
    truncations: list         # 4 leaves, then (12), (34)

    @property
    def ranks(self):
        return tuple(u.shape[1] for u in self.leaves) + (self.c12.shape[2], self.c34.shape[2])


def htucker_svd(t: np.ndarray, gamma: float) -> HTuckerFormat:
    """Alg. 2 H-Tucker-SVD for a 4D tensor.

    step 3: leaves by Alg. 1 with delta = gamma/sqrt(6) ||T||_F (reading Q8);
    step 4: W = T x_1 U1* x_2 U2* x_3 U3* x_4 U4* (projection by mode products,
            reading Q9, never a Kronecker matrix);
    steps 5-7: W12 = (r1 r2) x (r3 r4) matricisation, truncated SVD (delta as
            above) -> C12 = left vectors reshaped r1 x r2 x r12;
    step 8: the same for the (r3 r4) x (r1 r2) matricisation -> C34;
    steps 9-10: root C1234 = C12^H W12 conj(C34) (reading Q10), r12 x r34.
    """
    assert t.ndim == 4
    nrm = frob(t)
    tk = tucker_svd(t, gamma, n_trunc=6, norm=nrm)
    w = tk.core
    r1, r2, r3, r4 = w.shape
    delta = gamma / math.sqrt(6) * nrm
    w12 = np.reshape(w, (r1 * r2, r3 * r4), order="F")
    u12, s12, _ = svd(w12)
    tr12 = tail_rank(s12, delta)
    c12m = u12[:, :tr12.rank]
    w34 = w12.T
    u34, s34, _ = svd(w34)
    tr34 = tail_rank(s34, delta)
    c34m = u34[:, :tr34.rank]
    root = c12m.conj().T @ w12 @ c34m.conj()
    return HTuckerFormat(
        leaves=tk.factors,
        c12=np.reshape(c12m, (r1, r2, tr12.rank), order="F"),
        c34=np.reshape(c34m, (r3, r4, tr34.rank), order="F"),
        c1234=root,
        truncations=tk.truncations + [tr12, tr34],
    )
