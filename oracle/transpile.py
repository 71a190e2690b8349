"""ORACLE (test infrastructure only): basis-gate rewriting of an HHL gate list.

PAPER.md:68 (§I): "the HHL circuit that only solves a random 2-by-2 linear system ... already has
120 one-qubit gates and 90 two-qubit gates" -- the Qiskit-transpiled form of the circuit, whose gate
fusion (Fig. 4) SV-Sim reduces to 67 gates. This module produces the
same kind of stream from the oracle's own logical HHL list (oracle/hhl.py): only one-qubit gates
(2x2 dense, or 1-qubit diagonal phases) and CNOTs, by the textbook decompositions

* controlled-U (one control, 2x2 U): U = e^{i a} Rz(b) Ry(c) Rz(d), A = Rz(b) Ry(c/2),
  B = Ry(-c/2) Rz(-(d+b)/2), C = Rz((d-b)/2):  C-U = P(a)_ctrl · A · CX · B · CX · C   (Nielsen &
  Chuang Cor. 4.2 / Fig. 4.6);
* CP(t) (diagonal(1,1,1,e^{it})): P(t/2)_a · CX · P(-t/2)_b · CX · P(t/2)_b;
* SWAP: three CNOTs;
* the reciprocal rotation (an RY on the ancilla multiplexed by k clock qubits, angle 2 asin(s_m)):
  the Gray-code uniformly-controlled rotation (Mottonen et al. 2004): 2^k RY + 2^k CNOT with
  alpha = M^-1 theta, M_mi = (-1)^{popcount(m & gray(i))};
* H, U_b (2x2 for a 1-qubit system): kept as one-qubit gates.
Every decomposition is exact (no global phase is dropped), so the rewritten list applied by the oracle
equals the logical list's state to rounding (pinned in tests/test_oracle_pins.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import sim

X = np.array([[0, 1], [1, 0]], dtype=complex)


def rz(t):
    return np.array([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]], dtype=complex)


def ry(t):
    c, s = math.cos(t / 2), math.sin(t / 2)
    return np.array([[c, -s], [s, c]], dtype=complex)


def _one(q, U):
    return {"kind": "dense", "targets": [q], "data": np.asarray(U, dtype=complex)}


def _phase(q, t):
    return {"kind": "diagonal", "targets": [q], "data": np.array([1.0, np.exp(1j * t)])}


def _cx(c, t):
    return {"kind": "controlled", "targets": [t], "controls": [c], "cvals": 1, "data": X.copy()}


def zyz(U):
    """U = e^{i a} Rz(b) Ry(c) Rz(d) for a 2x2 unitary U."""
    det = np.linalg.det(U)
    a = np.angle(det) / 2
    V = U * np.exp(-1j * a)                          # SU(2)
    c = 2 * math.atan2(abs(V[1, 0]), abs(V[0, 0]))
    if abs(V[0, 0]) > 1e-12 and abs(V[1, 0]) > 1e-12:
        bp = np.angle(V[1, 1]) * 2                  # b + d
        bm = np.angle(V[1, 0]) * 2                  # b - d
        b, d = (bp + bm) / 2, (bp - bm) / 2
    elif abs(V[1, 0]) <= 1e-12:
        b, d = np.angle(V[1, 1]) * 2, 0.0
    else:
        b, d = np.angle(V[1, 0]) * 2, 0.0
    W = np.exp(1j * a) * rz(b) @ ry(c) @ rz(d)
    if np.abs(W - U).max() > 1e-9:                   # branch of the half-angles: fix the sign via a
        a += math.pi
        W = np.exp(1j * a) * rz(b) @ ry(c) @ rz(d)
    assert np.abs(W - U).max() < 1e-9
    return a, b, c, d


def controlled_1q(c, t, U):
    a, b, cc, d = zyz(U)
    A = rz(b) @ ry(cc / 2)
    B = ry(-cc / 2) @ rz(-(d + b) / 2)
    C = rz((d - b) / 2)
    return [_one(t, C), _cx(c, t), _one(t, B), _cx(c, t), _one(t, A), _phase(c, a)]


def cphase(a, b, t):
    return [_phase(a, t / 2), _cx(a, b), _phase(b, -t / 2), _cx(a, b), _phase(b, t / 2)]


def swap(a, b):
    return [_cx(a, b), _cx(b, a), _cx(a, b)]


def gray(i):
    return i ^ (i >> 1)


def multiplexed_ry(controls, target, thetas):
    """RY(thetas[m]) on target for control value m (bit j of m = controls[j])."""
    k = len(controls)
    N = 1 << k
    # control value m sees theta_m = sum_i (-1)^{popcount(m & gray(i))} alpha_i: before step i the CNOTs
    # have toggled the target's X conjugation for the controls in gray(i), and X Ry(a) X = Ry(-a)
    M = np.array([[(-1) ** bin(m & gray(i)).count("1") for i in range(N)] for m in range(N)], dtype=float)
    alpha = np.linalg.solve(M, np.asarray(thetas, dtype=float))
    out = []
    for i in range(N):
        out.append(_one(target, ry(alpha[i])))
        diff = gray(i) ^ gray((i + 1) % N)
        j = diff.bit_length() - 1                   # the control whose bit flips next (cyclic)
        out.append(_cx(controls[j], target))
    return out


def transpile(gates) -> list:
    """One-qubit + CNOT rewriting of an oracle HHL gate list (see module docstring)."""
    out = []
    for g in gates:
        k = g["kind"]
        if k == "dense" and len(g["targets"]) == 1:
            out.append(_one(g["targets"][0], g["data"]))
        elif k == "controlled" and len(g["targets"]) == 1 and len(g["controls"]) == 1 and g.get("cvals", 1) == 1:
            out += controlled_1q(g["controls"][0], g["targets"][0], np.asarray(g["data"], dtype=complex))
        elif k == "diagonal" and len(g["targets"]) == 2:
            d = np.asarray(g["data"], dtype=complex)
            assert abs(d[0] - 1) < 1e-15 and abs(d[1] - 1) < 1e-15 and abs(d[2] - 1) < 1e-15
            out += cphase(g["targets"][0], g["targets"][1], float(np.angle(d[3])))
        elif k == "swap":
            out += swap(*g["targets"])
        elif k == "recip_ry":
            clock = list(g["controls"])
            nc = len(clock)
            th = [2 * math.asin(sim.recip_s(m, nc, g["delta"], g.get("signed", 1), g.get("snap", 0.0)))
                  for m in range(1 << nc)]
            out += multiplexed_ry(clock, g["targets"][0], th)
        else:
            raise ValueError(f"no basis rewriting for {k} on {len(g['targets'])} targets")
    return out


def counts(gates):
    one = sum(1 for g in gates if len(g["targets"]) + len(g.get("controls", [])) == 1)
    return one, len(gates) - one
