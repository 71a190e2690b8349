"""ORACLE (test infrastructure only): the oracle's own HHL circuit builder + recovery.

Follows PAPER.md's "Practical HHL procedures" box (§III-A),
the conceptual circuit of Fig. 5 and the resources formula
(§III-B), with the qlsarepo/Qiskit settings the paper defers
to ("Following the settings in [qlsarepo]") as reconstructed in
SURVEY.md §8(c). Every garbled/silent point takes the reading listed in
DESIGN.md §Readings (R1..R17); the comments cite them.

Register layout (R1): system qubits 0..n_b-1 | clock qubits n_b..n_b+n_c-1
(clock value m = sum_j m_j 2^j, LSB first) | rotation ancilla n-1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import sim


@dataclass
class HHLPlan:
    A: np.ndarray           # padded system matrix, N×N
    b_hat: np.ndarray       # normalised, padded RHS
    b_norm: float
    n_orig: int
    n_b: int
    n_c: int
    n: int
    lam: np.ndarray         # eigenvalues of A (ascending, from eigh)
    V: np.ndarray           # eigenvectors (columns)
    lam_min: float          # min |lambda|
    lam_max: float          # max |lambda|
    kappa: float
    delta: float
    t: float
    phi: np.ndarray         # phi_s = lambda_s t / (2 pi)
    snap: float
    gates: list = field(default_factory=list)
    x_offset: int = 0       # Hermitian embedding: the solution sits in the lower half


def pad_system(A, b):
    """PAPER.md:167 step 1(b) "expand it to the nearest power of 2": identity padding of A,
    zero padding of b (R9)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n0 = A.shape[0]
    nb = max(1, math.ceil(math.log2(n0))) if n0 > 1 else 1
    N = 1 << nb
    Ap = np.eye(N)
    Ap[:n0, :n0] = A
    bp = np.zeros(N)
    bp[:n0] = b
    return Ap, bp, nb


def clock_qubits_default(n_b: int, kappa: float) -> int:
    """n_QPE per PAPER.md:234 read per F3/R2-R3: max(n_data+1, ceil(log2(kappa+1))) + 1 sign qubit."""
    return max(n_b + 1, math.ceil(math.log2(kappa + 1.0))) + 1


def get_delta(n_l: int, lam_min: float, lam_max: float) -> float:
    """qlsarepo _get_delta (R4): floor(lam_min (2^n_l - 1)/lam_max) / 2^n_l, snapping to 1 within 1e-7."""
    lt = abs(lam_min * (2 ** n_l - 1) / lam_max)
    if abs(lt - 1.0) < 1e-7:
        lt = 1.0
    return int(lt) / 2 ** n_l


def householder_prep(b_hat: np.ndarray) -> np.ndarray:
    """State preparation U_b with U_b|0> = |b> (R11): U_b = I - 2 v v^T/(v^T v), v = e0 - b_hat."""
    N = b_hat.size
    v = -b_hat.copy()
    v[0] += 1.0
    vv = float(v @ v)
    if vv < 1e-300:
        return np.eye(N, dtype=complex)
    return (np.eye(N) - 2.0 * np.outer(v, v) / vv).astype(complex)


def H1():
    return np.array([[1, 1], [1, -1]], dtype=complex) / math.sqrt(2.0)


def cp_diag(theta: float) -> np.ndarray:
    """CP(theta) = diag(1, 1, 1, e^{i theta}) (symmetric in its two qubits)."""
    return np.array([1, 1, 1, np.exp(1j * theta)], dtype=complex)


def qft_gates(qubits, inverse: bool = False) -> list:
    """Textbook QFT on `qubits` (qubits[0] = LSB of the register value), with swaps (R12):
    QFT|k> = N^-1/2 sum_m e^{+2 pi i k m / N}|m>. The inverse is the reversed list with
    conjugated phases."""
    q = list(qubits)
    n = len(q)
    gl = []
    for j in reversed(range(n)):
        gl.append({"kind": "dense", "targets": [q[j]], "data": H1()})
        for k in reversed(range(j)):
            gl.append({"kind": "diagonal", "targets": [q[j], q[k]], "data": cp_diag(math.pi / 2 ** (j - k))})
    for i in range(n // 2):
        gl.append({"kind": "swap", "targets": [q[i], q[n - 1 - i]]})
    if inverse:
        inv = []
        for g in reversed(gl):
            g2 = dict(g)
            if g["kind"] == "diagonal":
                g2["data"] = np.conj(g["data"])
            inv.append(g2)
        gl = inv
    return gl


def controlled_evolution(V, phi, j):
    """U_j = U^{2^j} = V diag(exp(2 pi i frac(2^j phi_s))) V^T (R13: frac(2^j phi) is exact in fp64)."""
    x = np.ldexp(phi, j)
    f = x - np.floor(x)
    return (V * np.exp(2j * np.pi * f)[None, :]) @ V.conj().T


def hermitize(Ap, bp):
    """PAPER.md:168-183 step 1(c): [[0, A], [A^T, 0]] [0; x] = [b; 0] (real A: A^dagger = A^T)."""
    N = Ap.shape[0]
    H = np.zeros((2 * N, 2 * N))
    H[:N, N:] = Ap
    H[N:, :N] = Ap.T
    return H, np.concatenate([bp, np.zeros(N)])


def plan(A, b, clock_qubits: int | None = None, snap: float = 1e-5) -> HHLPlan:
    """Steps 1-2 of the procedure box: normalise b, pad (step 1b), Hermitize a non-symmetric A
    (step 1c, after the expansion as Table 1's 30-bus* n_data = 6 implies), eigen-analyse,
    choose n_c, delta, t."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        raise ValueError("zero b")
    n0 = A.shape[0]
    Ap, bp, nb = pad_system(A, b)
    x_offset = 0
    if not np.allclose(Ap, Ap.T, atol=1e-10, rtol=0):
        x_offset = Ap.shape[0]
        Ap, bp = hermitize(Ap, bp)
        nb += 1
    lam, V = np.linalg.eigh(Ap)
    alam = np.abs(lam)
    lam_min, lam_max = float(alam.min()), float(alam.max())
    kappa = lam_max / lam_min
    nc = clock_qubits_default(nb, kappa) if not clock_qubits else int(clock_qubits)
    n_l = nc - 1                       # R3: sign qubit always present
    delta = get_delta(n_l, lam_min, lam_max)
    if delta == 0.0:
        raise ValueError("clock register too small (delta = 0)")
    t = 2.0 * math.pi * delta / lam_min / 2.0      # qlsarepo evolution time with neg_vals (R4)
    phi = (lam / lam_min) * (delta / 2.0)          # = lambda t / (2 pi), lam_min -> delta/2 exactly (R13)
    p = HHLPlan(A=Ap, b_hat=bp / bn, b_norm=bn, n_orig=n0, n_b=nb, n_c=nc, n=nb + nc + 1, lam=lam, V=V,
                lam_min=lam_min, lam_max=lam_max, kappa=kappa, delta=delta, t=t, phi=phi, snap=snap,
                x_offset=x_offset)
    return p


def build(p: HHLPlan) -> list:
    """Logical HHL gate list of Fig. 5:
    prep U_b; H^{⊗n_c}; c-U_j (j ascending); IQFT; RECIP_RY; QFT; c-U_j^† (j descending); H^{⊗n_c}.
    Count = n_c^2 + 5 n_c + 2 + 2 floor(n_c/2)."""
    nb, nc = p.n_b, p.n_c
    sys_q = list(range(nb))
    clk = [nb + j for j in range(nc)]
    anc = nb + nc
    g = [{"kind": "dense", "targets": sys_q, "data": householder_prep(p.b_hat)}]
    g += [{"kind": "dense", "targets": [q], "data": H1()} for q in clk]
    Us = [controlled_evolution(p.V, p.phi, j) for j in range(nc)]
    g += [{"kind": "controlled", "targets": sys_q, "controls": [clk[j]], "cvals": 1, "data": Us[j]}
          for j in range(nc)]
    g += qft_gates(clk, inverse=True)
    g.append({"kind": "recip_ry", "targets": [anc], "controls": clk, "delta": p.delta, "signed": 1,
              "snap": p.snap})
    g += qft_gates(clk, inverse=False)
    g += [{"kind": "controlled", "targets": sys_q, "controls": [clk[j]], "cvals": 1,
           "data": Us[j].conj().T.copy()} for j in reversed(range(nc))]
    g += [{"kind": "dense", "targets": [q], "data": H1()} for q in clk]
    p.gates = g
    return g


def postselect(psi: np.ndarray, p: HHLPlan):
    """Amplitudes with ancilla = 1 and clock = 0 (R7), P_succ = their squared norm."""
    base = 1 << (p.n - 1)
    sl = psi[base: base + (1 << p.n_b)].copy()
    return sl, float(np.sum(np.abs(sl) ** 2))


def recover(slice_amps: np.ndarray, p_succ: float, p: HHLPlan) -> np.ndarray:
    """PAPER.md:193-198 step 4 read per F3/R8: ||x|| = sqrt(P_succ)/lambda_min,
    x = ||x|| ||b|| |x>, |x> = slice/sqrt(P_succ); padding stripped (real part); for a Hermitized
    system the lower half is x."""
    if p_succ < 1e-12:
        raise ValueError("zero success probability")
    x_ket = slice_amps / math.sqrt(p_succ)
    x = (math.sqrt(p_succ) / p.lam_min) * p.b_norm * x_ket
    return np.real(x[p.x_offset: p.x_offset + p.n_orig])


def solve(A, b, clock_qubits=None, snap=1e-5):
    """Oracle HHL: plan, build, simulate the unfused list, post-select, recover."""
    p = plan(A, b, clock_qubits, snap)
    gates = build(p)
    psi = sim.run(gates, p.n)
    sl, ps = postselect(psi, p)
    return recover(sl, ps, p), ps, psi, p
