"""Pins for the CPU oracle (-m "not gpu"): values the paper prints, closed forms,
invariants, special cases and brute force — none of them re-calls the oracle's
own formula. A plausible mistake anywhere in oracle/ (dropped term, wrong sign,
wrong index, transposed operand) fails at least one of these.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import bruteforce as bf
from oracle import closed_form as cf
from oracle import hhl, sim
from workloads import configs, matpower, synthetic

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- single gates
def test_hadamard_on_zero():
    """S:136 H|0> = [1/sqrt2, 1/sqrt2] (textbook)."""
    psi = sim.run([{"kind": "dense", "targets": [0], "data": hhl.H1()}], 1)
    assert np.allclose(psi, [2 ** -0.5, 2 ** -0.5], atol=1e-15, rtol=0)


def test_bell_state_fig3():
    """PAPER.md:81 Fig. 3: H then CNOT on |00> -> (|00>+|11>)/sqrt2; 01 and 10 absent."""
    gold = _gold("fig3_bell.json")["probabilities"]
    cx = np.array([[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]], complex)   # control q0, target q1
    psi = sim.run([{"kind": "dense", "targets": [0], "data": hhl.H1()},
                   {"kind": "dense", "targets": [0, 1], "data": cx}], 2)
    probs = sim.marginal(psi, 2, [0, 1])
    for bits, p in gold.items():
        v = int(bits[1]) | (int(bits[0]) << 1)      # bitstring printed q1 q0
        assert abs(probs[v] - p) < 1e-15


def test_controlled_x_is_cnot():
    """A 'controlled' X with control q1, target q0 equals the textbook CNOT permutation."""
    X = np.array([[0, 1], [1, 0]], complex)
    for start in range(4):
        psi0 = np.zeros(4, complex)
        psi0[start] = 1
        out = sim.run([{"kind": "controlled", "targets": [0], "controls": [1], "cvals": 1, "data": X}], 2, psi0)
        expect = start ^ 1 if start & 2 else start
        assert abs(out[expect] - 1) < 1e-15


def test_cvals_zero_control():
    """Control value 0 fires on |0> of the control (negated control)."""
    X = np.array([[0, 1], [1, 0]], complex)
    out = sim.run([{"kind": "controlled", "targets": [1], "controls": [0], "cvals": 0, "data": X}], 2)
    assert abs(out[2] - 1) < 1e-15


# -------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(6))
def test_random_circuits_vs_bruteforce(seed):
    """S:138 random circuits vs the dense full-operator product (tensordot embedding), width ≤ 6."""
    n = 3 + seed % 4
    gates = synthetic.random_circuit(n, 25, seed=100 + seed, kmax=3)
    psi0 = synthetic.random_state(n, seed)
    a = sim.run(gates, n, psi0)
    b = bf.run(gates, n, psi0)
    assert np.abs(a - b).max() < 1e-13


def test_c1_full_circuit_unitary():
    """C1 (5 qubits, 28 gates): oracle state = first column of the brute-force circuit unitary,
    which is unitary to 1e-13."""
    A, b, nc = configs.get("C1")
    p = hhl.plan(A, b, nc)
    gates = hhl.build(p)
    assert len(gates) == 28
    U = bf.circuit_unitary(gates, p.n)
    assert np.abs(U @ U.conj().T - np.eye(32)).max() < 1e-13
    psi = sim.run(gates, p.n)
    assert np.abs(psi - U[:, 0]).max() < 1e-13


def test_recip_ry_vs_bruteforce():
    """Multiplexed RY with sign qubit on 1 ancilla + 4 clock qubits, vs block-diagonal operator."""
    g = {"kind": "recip_ry", "targets": [0], "controls": [1, 2, 3, 4], "delta": 3 / 8, "signed": 1, "snap": 0.0}
    psi0 = synthetic.random_state(5, 11)
    assert np.abs(sim.run([g], 5, psi0) - bf.run([g], 5, psi0)).max() < 1e-14


def test_marginal_consistency():
    """S:180 marginal over a subset = full distribution summed by those bits (numpy reshape)."""
    n = 7
    psi = synthetic.random_state(n, 3)
    full = np.abs(psi) ** 2
    m = sim.marginal(psi, n, [5, 1])
    T = full.reshape([2] * n)                   # axis a <-> qubit n-1-a
    ref = T.sum(axis=tuple(a for a in range(n) if a not in (n - 1 - 5, n - 1 - 1)))   # axes (q5, q1)
    # output index v = bit(q5) + 2 bit(q1); ref is indexed [q5, q1]
    assert np.allclose(m, [ref[0, 0], ref[1, 0], ref[0, 1], ref[1, 1]], atol=1e-15)
    assert abs(sim.marginal(psi, n, []).sum() - 1) < 1e-13


# ------------------------------------------------------------------ QFT / QPE
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_qft_is_dft(n):
    """Textbook QFT list = DFT matrix F[m,k] = e^{+2 pi i k m/N}/sqrt N (little-endian register)."""
    N = 1 << n
    F = np.exp(2j * np.pi * np.outer(np.arange(N), np.arange(N)) / N) / math.sqrt(N)
    U = bf.circuit_unitary(hhl.qft_gates(range(n)), n)
    assert np.abs(U - F).max() < 1e-13
    Ui = bf.circuit_unitary(hhl.qft_gates(range(n), inverse=True), n)
    assert np.abs(Ui - F.conj().T).max() < 1e-13


def _qpe_clock_distribution(A, s_idx, nc):
    """Run the oracle's QPE half (H layer, c-U_j, IQFT) on eigenvector s; return P(clock=m)."""
    p = hhl.plan(A, np.ones(A.shape[0]), nc)
    nb = p.n_b
    gates = hhl.build(p)
    q = gates[1: 1 + 2 * nc + nc + nc * (nc - 1) // 2 + nc // 2]     # H, cU, IQFT
    n = p.n
    psi0 = np.zeros(1 << n, complex)
    psi0[: 1 << nb] = p.V[:, s_idx]
    psi = sim.run(q, n, psi0)
    return sim.marginal(psi, n, list(range(nb, nb + nc))), p


@pytest.mark.parametrize("nc", [3, 4, 5])
def test_qpe_exact_on_representable_phase(nc):
    """representable eigenphase -> P(clock = m0) = 1 within 1e-12. A = diag(1, 3),
    lambda_min = 1 maps to m0 = delta 2^(nc-1) exactly, lambda = 3 to 3 m0."""
    A = np.diag([1.0, 3.0])
    for s in range(2):
        probs, p = _qpe_clock_distribution(A, s, nc)
        m0 = round(p.phi[s] * (1 << nc))
        assert abs(p.phi[s] * (1 << nc) - m0) < 1e-12
        assert probs[m0] > 1 - 1e-12


def test_qpe_fejer_kernel():
    """Non-representable phase: clock distribution = Fejér kernel sin^2(pi N d)/(N^2 sin^2(pi d)), d = phi - m/N."""
    A = np.diag([1.0, 2.7])
    nc = 5
    N = 1 << nc
    probs, p = _qpe_clock_distribution(A, 1, nc)
    phi = p.phi[1]
    m = np.arange(N)
    d = phi - m / N
    fejer = np.sin(np.pi * N * d) ** 2 / (N ** 2 * np.sin(np.pi * d) ** 2)
    assert np.abs(probs - fejer).max() < 1e-12


# ----------------------------------------------------------------- HHL oracle
def test_gate_count_formula():
    """n_c^2 + 5 n_c + 2 + 2 floor(n_c/2) gates (C1 28, C2 74, C3 162, C3p 114)."""
    for name, want in [("C1", 28), ("C2", 74), ("C3", 162), ("C3p", 114)]:
        A, b, nc = configs.get(name)
        assert len(hhl.build(hhl.plan(A, b, nc))) == want


def test_norm_preserved_every_gate():
    """S:177 norm preservation after every gate (1e-12) on C3 (15 qubits, 162 gates)."""
    A, b, nc = configs.get("C3")
    p = hhl.plan(A, b, nc)
    psi = sim.zero_state(p.n)
    for g in hhl.build(p):
        sim.apply_gate(psi, p.n, g)
        assert abs(np.vdot(psi, psi).real - 1) < 1e-12


def test_c1_exact():
    """C1: eigenvalues 1, 3 exactly representable -> P = 5/9, x = solve(A, b) = (2/3, 1/3)."""
    A, b, nc = configs.get("C1")
    x, ps, psi, p = hhl.solve(A, b, nc)
    assert p.n == 5 and p.delta == 0.25 and abs(p.t - math.pi / 4) < 1e-15
    assert abs(ps - 5 / 9) < 1e-12
    assert np.abs(x - np.linalg.solve(A, b)).max() < 1e-12
    assert np.abs(x - [2 / 3, 1 / 3]).max() < 1e-12


def test_identity_system():
    """S:314 A = I -> x = b."""
    b = np.array([3.0, 4.0, 0.0, -1.0])
    x, ps, _, _ = hhl.solve(np.eye(4), b)
    assert np.abs(x - b).max() < 1e-12


def test_diagonal_representable():
    """S:306 diagonal A with representable eigenvalues -> exact direct solve."""
    A = np.diag([1.0, 2.0])
    b = np.array([0.6, 0.8])
    x, _, _, _ = hhl.solve(A, b)
    assert np.abs(x - np.linalg.solve(A, b)).max() < 1e-12


def test_table1_14bus():
    """PAPER.md:289-296 Table 1, 14-bus: 13×13, kappa 119.2, n_total 13 = (4, 8), err 1.97e-3."""
    gold = _gold("table1.json")["14-bus"]
    A, b = matpower.case14()
    assert A.shape[0] == gold["matrix_size"]
    x, ps, psi, p = hhl.solve(A, b)              # default n_c from the resources formula (R2)
    assert 0 <= p.kappa - gold["kappa"] < 0.1          # printed truncated to 1 decimal (119.285 -> 119.2)
    assert (p.n, p.n_b, p.n_c) == (gold["n_total"], gold["n_data"], gold["n_qpe"])
    err = np.linalg.norm(x - np.linalg.solve(A, b))
    assert abs(err - gold["err_l2"]) < 0.005e-3


def test_table1_30bus():
    """PAPER.md:289-296 Table 1, 30-bus: 29×29, kappa 492.5, n_total 16 = (5, 10), err 1.18e-3."""
    gold = _gold("table1.json")["30-bus"]
    A, b = matpower.case30()
    assert A.shape[0] == gold["matrix_size"]
    x, ps, psi, p = hhl.solve(A, b)
    assert 0 <= p.kappa - gold["kappa"] < 0.1          # printed truncated to 1 decimal (119.285 -> 119.2)
    assert (p.n, p.n_b, p.n_c) == (gold["n_total"], gold["n_data"], gold["n_qpe"])
    err = np.linalg.norm(x - np.linalg.solve(A, b))
    assert abs(err - gold["err_l2"]) < 0.005e-3


def test_case5_eigenvalues():
    """Appendix A.2 checks (fixture sanity): eigenvalues 22.736, 59.281, 219.063, 368.014."""
    A, b = matpower.case5()
    lam = np.linalg.eigvalsh(A)
    assert np.allclose(lam, [22.736, 59.281, 219.063, 368.014], atol=2e-3)
    p = hhl.plan(A, b)
    assert p.n_c == 6


@pytest.mark.parametrize("name", ["C1", "C2", "C3p", "C3"])
def test_closed_form_full_state(name):
    """SURVEY eq. CF: every amplitude of the gate-level oracle equals the analytic state (≤ 1e-12)."""
    A, b, nc = configs.get(name)
    x, ps, psi, p = hhl.solve(A, b, nc)
    assert np.abs(psi - cf.full_state(p)).max() < 1e-12
    xt, P = cf.postselected(p)
    assert abs(P - ps) < 1e-12
    sl, _ = hhl.postselect(psi, p)
    assert np.abs(sl - xt).max() < 1e-12


def test_closed_form_sampled_matches_full():
    A, b, nc = configs.get("C3")
    p = hhl.plan(A, b, nc)
    idx = synthetic.rng(5).integers(0, 1 << p.n, 40)
    full = cf.full_state(p)
    assert np.abs(cf.sampled_amplitudes(p, idx) - full[idx]).max() < 1e-13


def test_closed_form_block_amplitudes_match_full():
    """block_amplitudes (high clock bits contracted by a matrix-vector product, low bits by a
    Walsh transform) = full_state on whole clock blocks, incl. block 0 (the post-selected slice)."""
    for name, b in (("C3", 8), ("C3", 0), ("C2", 6), ("C3p", 3)):
        A, bb, nc = configs.get(name)
        p = hhl.plan(A, bb, nc)
        full = cf.full_state(p).reshape(2, 1 << p.n_c, 1 << p.n_b)
        khs = [0, (1 << (p.n_c - b)) - 1, (1 << (p.n_c - b)) // 3]
        blk = cf.block_amplitudes(p, khs, b)
        for j, kh in enumerate(khs):
            assert np.abs(blk[:, j] - full[:, kh << b:(kh + 1) << b]).max() < 1e-13


def test_recip_table_matches_c_definition():
    """numpy s_m (closed_form) = C s_m (sv_oracle.c) incl. sign half, clipping and snapping."""
    for nc, delta, snap in [(3, 0.25, 0.0), (6, 1 / 32, 1e-5), (10, 1 / 128, 1e-5), (12, 0.3, 0.01)]:
        tab = cf.recip_table(nc, delta, 1, snap)
        for m in list(range(0, 1 << nc, max(1, (1 << nc) // 97))) + [1, (1 << (nc - 1)), (1 << nc) - 1]:
            assert tab[m] == sim.recip_s(m, nc, delta, 1, snap)
    # special values: s(m_min) = 1, s(0) = 0, negative half is the mirrored negative
    tab = cf.recip_table(6, 1 / 32, 1, 0.0)
    assert tab[1] == 1.0 and tab[0] == 0.0 and tab[2] == 0.5 and tab[64 - 2] == -0.5


def test_accuracy_improves_with_clock_register():
    """HHL post-selected state -> normalize(solve(A, b)) as the clock register grows (north_star)."""
    A, b = matpower.case5()
    xt = np.linalg.solve(A, b)
    xt /= np.linalg.norm(xt)
    errs = []
    for nc in (6, 8, 10):
        x, _, _, _ = hhl.solve(A, b, nc)
        errs.append(np.linalg.norm(x / np.linalg.norm(x) - xt))
    assert errs[0] > errs[1] > errs[2]
    assert errs[-1] < 5e-3


def test_alpha_geometric_equals_fft():
    """The geometric-series QPE amplitude (used at n_c > 16) equals the FFT of the phase vector."""
    for phi in (0.123456789, 0.25, 0.49999, 1 / 3):
        for nc in (4, 10, 14):
            a = cf.alpha_geometric(phi, nc)
            b = np.fft.fft(cf.phase_vector(phi, nc)) / (1 << nc)
            assert np.abs(a - b).max() < 1e-12          # FFT sums 2^nc rounded terms
            p2 = cf.alpha_abs2(phi, nc)
            assert np.abs(p2 - np.abs(b) ** 2).max() < 5e-12


def test_hermitian_embedding_exact():
    """[[0, A], [A^T, 0]] [0; x] = [b; 0]. A = [[0, 1], [3, 0]] has singular values
    1 and 3, so the embedded eigenvalues +-1, +-3 are representable (negative ones through the sign
    qubit) and HHL is exact: x = solve(A, b)."""
    A = np.array([[0.0, 1.0], [3.0, 0.0]])
    b = np.array([0.6, 0.8])
    x, ps, psi, p = hhl.solve(A, b)
    assert (p.n_b, p.x_offset) == (2, 2)
    assert sorted(np.round(p.lam, 12)) == [-3, -1, 1, 3]
    assert np.abs(x - np.linalg.solve(A, b)).max() < 1e-12
    # the upper half of the post-selected vector is 0 (the [0; x] structure)
    sl, _ = hhl.postselect(psi, p)
    assert np.abs(sl[:2]).max() < 1e-12


def test_hermitian_embedding_random():
    """A seeded non-symmetric 4x4 system: relative error shrinks with the clock register."""
    g = synthetic.rng(3)
    A = g.standard_normal((4, 4)) + 4 * np.eye(4)
    b = g.standard_normal(4)
    xt = np.linalg.solve(A, b)
    errs = [np.linalg.norm(hhl.solve(A, b, nc)[0] - xt) / np.linalg.norm(xt) for nc in (6, 8, 10)]
    assert errs[0] > errs[2] and errs[2] < 5e-3


@pytest.mark.parametrize("name", ["C1"])
def test_transpiled_hhl_stream_equals_logical(name):
    """oracle/transpile.py: the one-qubit + CNOT rewriting of the HHL list (PAPER.md:68's transpiled
    form) is exact: same final state as the logical list (no dropped global phase), CNOTs and 1q only."""
    from oracle import transpile as tr
    A, b, nc = configs.get(name)
    p = hhl.plan(A, b, nc)
    g = hhl.build(p)
    t = tr.transpile(g)
    one, two = tr.counts(t)
    assert one + two == len(t) and two > 0
    assert all(len(x["targets"]) + len(x.get("controls", [])) <= 2 for x in t)
    assert np.abs(sim.run(g, p.n) - sim.run(t, p.n)).max() < 1e-12


def test_multiplexed_ry_bruteforce():
    """Gray-code uniformly-controlled RY vs the direct multiplexed matrix (random angles, 3 controls)."""
    from oracle import transpile as tr
    g = synthetic.rng(9)
    th = g.uniform(-3, 3, 8)
    n = 4
    psi0 = synthetic.random_state(n, 2)
    ref = psi0.copy()
    for i in range(1 << n):
        if (i >> 3) & 1:
            continue
        m = i & 7
        c, s = np.cos(th[m] / 2), np.sin(th[m] / 2)
        a0, a1 = ref[i], ref[i | 8]
        ref[i], ref[i | 8] = c * a0 - s * a1, s * a0 + c * a1
    assert np.abs(sim.run(tr.multiplexed_ry([0, 1, 2], 3, th), n, psi0) - ref).max() < 1e-13
