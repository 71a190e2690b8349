"""ORACLE (test infrastructure only): closed-form HHL final state (SURVEY §8(c) eq. CF).

An analytic pin on the gate-level oracle, derived independently of it: for the
textbook circuit (H layer, c-U^{2^j}, IQFT, reciprocal RY, QFT, c-U^{2^j}†, H
layer) and |b> = sum_s beta_s |v_s>,

    alpha_m(phi) = N_c^-1 sum_k e^{2 pi i k (phi - m/N_c)}        (QPE amplitude)
    psi[a, k, .] = sum_s beta_s v_s · y_{s,a}[k],
    y_{s,a} = H^{⊗n_c} · diag(e^{-2 pi i phi_s k}) · F · (r_a ⊙ alpha(phi_s)),
    F|m> = N_c^-1/2 sum_k e^{+2 pi i k m/N_c}|k>,  r_1 = s, r_0 = sqrt(1 - s^2),

and the post-selected vector x~ = sum_s beta_s v_s sum_m |alpha_m(phi_s)|^2 s_m
with P_succ = ||x~||^2. The phases e^{2 pi i phi k} are formed as products of
e^{2 pi i frac(2^j phi)} over the set bits of k (R13), like the circuit does.

The reciprocal s_m is re-derived here from its definition
vectorised in numpy; tests/test_oracle_pins.py checks it against sv_oracle.c.
"""
from __future__ import annotations

import numpy as np

try:                                   # multi-threaded FFT for the 2^25-point transforms at S30
    import scipy.fft as _fft

    def _ifft(x):
        return _fft.ifft(x, workers=-1)
except Exception:                      # pragma: no cover
    _ifft = np.fft.ifft


def recip_table(n_c: int, delta: float, signed: int = 1, snap: float = 0.0) -> np.ndarray:
    """s_m for m = 0..2^n_c - 1 (definition in SURVEY §8(a) a7 / DESIGN.md R6)."""
    Nc = 1 << n_c
    m = np.arange(Nc, dtype=np.float64)
    sign = np.ones(Nc)
    mp = m.copy()
    if signed:
        neg = np.arange(Nc) >= (Nc >> 1)
        mp[neg] = Nc - m[neg]
        sign[neg] = -1.0
    L = 2.0 ** (n_c - (1 if signed else 0))
    with np.errstate(divide="ignore"):
        r = np.where(mp > 0, delta * L / np.where(mp > 0, mp, 1.0), np.inf)
    s = np.where(np.abs(r - 1.0) <= snap, 1.0, np.where(r < 1.0, r, 0.0))
    s[0] = 0.0
    return sign * s


def phase_vector(phi: float, n_c: int) -> np.ndarray:
    """e^{2 pi i phi k} for k < 2^n_c, as prod_j e^{2 pi i frac(2^j phi)}^{k_j}."""
    ph = np.ones(1, dtype=np.complex128)
    for j in range(n_c):
        x = np.ldexp(phi, j)
        f = x - np.floor(x)
        ph = np.concatenate([ph, ph * np.exp(2j * np.pi * f)])
    return ph


def alpha_geometric(phi: float, n_c: int) -> np.ndarray:
    """alpha_m(phi) for all m by the geometric series N^-1 (e^{2 pi i N d} - 1)/(e^{2 pi i d} - 1),
    d = phi - m/N, with e^{2 pi i N d} = e^{2 pi i frac(N phi)} and e^{2 pi i d} - 1 =
    2i sin(pi d) e^{i pi d}. phi - m/N is exact near the peak (Sterbenz), so this is accurate
    where alpha is large. Equal to fft(phase_vector)/N (pinned in tests)."""
    Nc = 1 << n_c
    d = phi - np.arange(Nc, dtype=np.float64) / Nc
    x = np.ldexp(phi, n_c)
    F = x - np.floor(x)
    num = complex(np.cos(2 * np.pi * F) - 1.0, np.sin(2 * np.pi * F))
    pd = np.pi * d
    sd = np.sin(pd)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / (2.0 * Nc * sd)
    # num / (2i sd e^{i pi d} N) = num * (-i) e^{-i pi d} / (2 sd N)
    w = num * -1j
    with np.errstate(invalid="ignore"):
        a = (w * inv) * (np.cos(pd) - 1j * sd)
    a[sd == 0.0] = 1.0
    return a


def alpha_abs2(phi: float, n_c: int) -> np.ndarray:
    """|alpha_m(phi)|^2 = sin^2(pi N d) / (N^2 sin^2(pi d)) (Fejér kernel), sin(pi N d) = ±sin(pi frac(N phi))."""
    Nc = 1 << n_c
    d = phi - np.arange(Nc, dtype=np.float64) / Nc
    x = np.ldexp(phi, n_c)
    sF = np.sin(np.pi * (x - np.floor(x)))
    sd = np.sin(np.pi * d)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = (sF / Nc) ** 2 / (sd * sd)
    r[sd == 0.0] = 1.0
    return r


def fwht(v: np.ndarray) -> np.ndarray:
    """Normalised Walsh–Hadamard transform H^{⊗n} v (little-endian, any bit order is the same)."""
    v = v.copy()
    n = v.size
    h = 1
    while h < n:
        v = v.reshape(-1, 2, h)
        a = v[:, 0, :].copy()
        b = v[:, 1, :]
        v[:, 0, :] = a + b
        v[:, 1, :] = a - b
        v = v.reshape(n)
        h *= 2
    return v / np.sqrt(n)


def _y_vectors(phi: float, n_c: int, s_tab: np.ndarray):
    Nc = 1 << n_c
    ph = phase_vector(phi, n_c)
    alpha = alpha_geometric(phi, n_c) if n_c > 16 else np.fft.fft(ph) / Nc                      # alpha_m = N^-1 sum_k e^{2 pi i k phi} e^{-2 pi i k m/N}
    r1 = s_tab
    r0 = np.sqrt(1.0 - s_tab ** 2)
    out = []
    for r in (r0, r1):
        z = _ifft(r * alpha) * np.sqrt(Nc)       # F (r ⊙ alpha)
        out.append(np.conj(ph) * z)                    # controlled-U^† phases, before the final H layer
    return out


def full_state(p) -> np.ndarray:
    """Whole 2^n state vector for an oracle.hhl.HHLPlan (n_c <= ~20)."""
    nb, nc = p.n_b, p.n_c
    Nc = 1 << nc
    N = 1 << nb
    s_tab = recip_table(nc, p.delta, 1, p.snap)
    beta = p.V.T @ p.b_hat
    psi = np.zeros((2, Nc, N), dtype=np.complex128)      # [ancilla, clock, sys]
    for s in range(N):
        if beta[s] == 0.0:
            continue
        w0, w1 = _y_vectors(p.phi[s], nc, s_tab)
        y0, y1 = fwht(w0), fwht(w1)
        psi[0] += beta[s] * np.outer(y0, p.V[:, s])
        psi[1] += beta[s] * np.outer(y1, p.V[:, s])
    return psi.reshape(-1)


def postselected(p):
    """x~ = sum_s beta_s v_s sum_m |alpha_m(phi_s)|^2 s_m and P_succ = ||x~||^2."""
    nc = p.n_c
    Nc = 1 << nc
    s_tab = recip_table(nc, p.delta, 1, p.snap)
    beta = p.V.T @ p.b_hat
    x = np.zeros(p.A.shape[0])
    for s in range(beta.size):
        a2 = alpha_abs2(p.phi[s], nc) if nc > 16 else np.abs(np.fft.fft(phase_vector(p.phi[s], nc)) / Nc) ** 2
        x += beta[s] * p.V[:, s] * float(np.sum(a2 * s_tab))
    return x, float(x @ x)


def sampled_amplitudes(p, indices) -> np.ndarray:
    """psi[i] for selected logical indices i, for any n_c (cost O(N · 2^n_c) per eigen-component
    plus O(2^n_c) per distinct clock value): the Walsh row of clock value k is contracted bit by bit."""
    nb, nc = p.n_b, p.n_c
    idx = np.asarray(indices, dtype=np.int64)
    sys_i = idx & ((1 << nb) - 1)
    k_i = (idx >> nb) & ((1 << nc) - 1)
    a_i = (idx >> (nb + nc)) & 1
    ks = np.unique(k_i)
    s_tab = recip_table(nc, p.delta, 1, p.snap)
    beta = p.V.T @ p.b_hat
    Nc = 1 << nc
    yk = np.zeros((2, ks.size, beta.size), dtype=np.complex128)   # y_{s,a}[k]
    for s in range(beta.size):
        if beta[s] == 0.0:
            continue
        ws = _y_vectors(p.phi[s], nc, s_tab)
        for a in (0, 1):
            for ki, k in enumerate(ks):
                v = ws[a]
                for j in range(nc):                 # contract bit j (LSB first) with (1, (-1)^{k_j})
                    v = v.reshape(-1, 2)
                    v = v[:, 0] + v[:, 1] if not ((int(k) >> j) & 1) else v[:, 0] - v[:, 1]
                yk[a, ki, s] = v[0] / np.sqrt(Nc)
    out = np.empty(idx.size, dtype=np.complex128)
    kpos = {int(k): i for i, k in enumerate(ks)}
    for t in range(idx.size):
        y = yk[a_i[t], kpos[int(k_i[t])]]
        out[t] = np.sum(beta * y * p.V[sys_i[t], :])
    return out


def block_amplitudes(p, k_highs, b: int) -> np.ndarray:
    """psi over whole clock blocks: for each k_high in k_highs, every clock value
    k = k_high·2^b + k_low (k_low < 2^b), every system index and both ancilla values.
    Returns psi_blk[a, j, k_low, sys] = psi[sys + 2^n_b·(k_high_j·2^b + k_low) + 2^(n-1)·a].

    Same eq. CF as full_state; the final H^{⊗n_c} row of k is split as
    (-1)^{k·m} = (-1)^{k_high·m_high} (-1)^{k_low·m_low}: the high bits are contracted with one
    matrix-vector product per block (O(2^n_c)), the low bits by a 2^b-point Walsh transform.
    Cost per eigen-component: the two 2^n_c-point transforms of _y_vectors plus one pass per block."""
    nb, nc = p.n_b, p.n_c
    Nc = 1 << nc
    N = 1 << nb
    if not 0 <= b <= nc:
        raise ValueError("block bits out of range")
    nh = nc - b
    s_tab = recip_table(nc, p.delta, 1, p.snap)
    beta = p.V.T @ p.b_hat
    out = np.zeros((2, len(k_highs), 1 << b, N), dtype=np.complex128)
    # Walsh rows of the high bits: sign[j, m_high] = (-1)^{popcount(k_high_j & m_high)}
    mh = np.arange(1 << nh, dtype=np.int64)
    signs = np.empty((len(k_highs), 1 << nh))
    for j, kh in enumerate(k_highs):
        x = np.bitwise_and(mh, int(kh))
        par = np.zeros(mh.size, dtype=np.int64)
        while np.any(x):
            par ^= x & 1
            x >>= 1
        signs[j] = 1.0 - 2.0 * par
    for s in range(beta.size):
        if beta[s] == 0.0:
            continue
        ws = _y_vectors(p.phi[s], nc, s_tab)
        for a in (0, 1):
            W = ws[a].reshape(1 << nh, 1 << b)          # m = m_low + 2^b m_high
            U = signs @ W                               # (blocks, 2^b): high bits contracted
            for j in range(len(k_highs)):
                y = fwht(U[j]) * np.sqrt(1 << b) / np.sqrt(Nc)   # unnormalised low-bit Walsh, / sqrt(N_c)
                out[a, j] += beta[s] * np.outer(y, p.V[:, s])
    return out
