"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle, element by element.

Bar (north_star): max-abs amplitude error <= 1e-10, identical
post-selection index sets, |dP| <= 1e-12. Kernel-level cases use 1e-12.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2402_08136_b200 as pkg
from oracle import closed_form as cf
from oracle import hhl as ohhl
from oracle import sim
from workloads import configs, synthetic

pytestmark = pytest.mark.gpu

MODES = [dict(tile_qubits=-1), dict(tile_qubits=6, tile_jit=-1), dict(tile_qubits=10, tile_jit=-1),
         dict(tile_qubits=9, tile_jit=1)]


def run_both(n, gates, psi0=None, fused=True, **kw):
    st = pkg.State(n)
    if psi0 is not None:
        st.write(psi0)
    if fused:
        st.apply_circuit(gates, **kw)
    else:
        st.apply_fused(gates)
    got = st.read()
    ref = sim.run(gates, n, psi0)
    return got, ref, st


def placements(n, k, g):
    yield list(range(k))                                  # low bits (coalescing hazard)
    yield list(range(n - k, n))                           # top bits
    mid = n // 2 - k // 2
    yield list(range(mid, mid + k))
    yield [int(x) for x in g.permutation(n)[:k]]          # split, unsorted order


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_dense_every_placement(k, mode):
    n = 11
    g = synthetic.rng(10 + k)
    for t in placements(n, k, g):
        gates = [{"kind": "dense", "targets": t, "data": synthetic.haar_unitary(k, g)}]
        got, ref, _ = run_both(n, gates, synthetic.random_state(n, k), fusion_kmax=0, **mode)
        assert np.abs(got - ref).max() < 1e-12, (k, t)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k,c", [(1, 1), (2, 2), (4, 1), (3, 3), (5, 2)])
def test_controlled(k, c, mode):
    n = 12
    g = synthetic.rng(100 + 10 * k + c)
    for trial in range(4):
        q = [int(x) for x in g.permutation(n)[: k + c]]
        gates = [{"kind": "controlled", "targets": q[:k], "controls": q[k:], "cvals": int(g.integers(1 << c)),
                  "data": synthetic.haar_unitary(k, g)}]
        got, ref, _ = run_both(n, gates, synthetic.random_state(n, trial), fusion_kmax=0, **mode)
        assert np.abs(got - ref).max() < 1e-12, (k, c, q)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", [1, 2, 5, 9, 12])
def test_diagonal(k, mode):
    n = 13
    g = synthetic.rng(200 + k)
    for t in placements(n, k, g):
        gates = [{"kind": "diagonal", "targets": t, "data": synthetic.random_phases(k, g)}]
        got, ref, _ = run_both(n, gates, synthetic.random_state(n, k), fusion_kmax=0, **mode)
        assert np.abs(got - ref).max() < 1e-12, (k, t)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("signed,snap", [(1, 0.0), (1, 1e-5), (0, 0.0), (1, 0.2)])
def test_recip_ry(signed, snap, mode):
    n = 12
    g = synthetic.rng(300)
    for anc, clock in [(11, list(range(1, 11))), (0, list(range(4, 12))), (5, [9, 1, 7, 3, 11]),
                       (11, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10])]:
        nc = len(clock)
        delta = float(g.integers(1, 1 << (nc - 1))) / 2 ** (nc - 1)
        gates = [{"kind": "recip_ry", "targets": [anc], "controls": clock, "delta": delta, "signed": signed,
                  "snap": snap}]
        got, ref, _ = run_both(n, gates, synthetic.random_state(n, anc), fusion_kmax=0, **mode)
        assert np.abs(got - ref).max() < 1e-12, (anc, clock)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("kmax", [0, 2, 3, 4, 5])
def test_random_circuits_fused(kmax, mode):
    """Fusion transparency: fused + scheduled circuit = unfused oracle, width 10-14."""
    for seed in range(3):
        n = 10 + 2 * seed
        gates = synthetic.random_circuit(n, 120, seed=seed + 1000 * kmax, kmax=3)
        got, ref, st = run_both(n, gates, synthetic.random_state(n, seed), fusion_kmax=kmax, **mode)
        assert np.abs(got - ref).max() < 1e-10
        assert abs(st.norm2() - 1.0) < 1e-12


def test_apply_fused_matches():
    n = 9
    gates = synthetic.random_circuit(n, 40, seed=5, kmax=4)
    got, ref, _ = run_both(n, gates, synthetic.random_state(n, 5), fused=False)
    assert np.abs(got - ref).max() < 1e-12


def test_basis_gate_stream_paper_fusion():
    """Paper-mode fusion (k_max = 2, Fig. 4) on a transpiled-style 1q/CX stream."""
    n = 5
    gates = synthetic.basis_circuit(n, 210, seed=7)
    got, ref, _ = run_both(n, gates, None, fusion_kmax=2, tile_qubits=-1)
    assert np.abs(got - ref).max() < 1e-10


@pytest.mark.parametrize("name", ["C1", "C2", "C3p", "C3"])
@pytest.mark.parametrize("opts", [dict(), dict(tile_qubits=-1), dict(fusion_kmax=-1, tile_qubits=-1),
                                  dict(fusion_kmax=2, tile_qubits=8), dict(init_fold=-1), dict(qpe_mode=1),
                                  dict(qpe_mode=1, tile_qubits=-1), dict(qpe_mode=1, fusion_kmax=1, tile_qubits=11),
                                  dict(qpe_mode=1, fusion_kmax=1, tile_qubits=10, tile_jit=1),
                                  dict(fusion_kmax=2, tile_qubits=10, tile_jit=1)])
def test_hhl_configs_full_state(name, opts):
    """C1-C3 (configs[0..2]) + C3p (Table 1 14-bus): every amplitude within 1e-10 of the oracle,
    identical post-selection index set, |dP| <= 1e-12, x within 1e-10."""
    A, b, nc = configs.get(name)
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    st = pkg.State(p.n)
    prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, **opts)
    prog.run()
    psi = st.read()
    assert np.abs(psi - psi_o).max() < 1e-10
    x, ps = prog.readout()
    assert abs(ps - po) < 1e-12
    assert np.abs(x - xo).max() < 1e-10
    fq = list(range(p.n_b, p.n_b + p.n_c)) + [p.n - 1]
    fv = [0] * p.n_c + [1]
    amps, idx, pp = st.postselect_slice(fq, fv)
    base = 1 << (p.n - 1)
    assert list(idx) == list(range(base, base + (1 << p.n_b)))
    assert np.abs(amps - psi_o[base: base + (1 << p.n_b)]).max() < 1e-10


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_hhl_solve_end_to_end(name):
    A, b, nc = configs.get(name)
    xo, po, _, p = ohhl.solve(A, b, nc)
    x, rep = pkg.hhl_solve(A, b, clock_qubits=nc)
    assert (rep["n_data"], rep["n_clock"], rep["n_total"]) == (p.n_b, p.n_c, p.n)
    assert abs(rep["p_success"] - po) < 1e-12
    assert abs(rep["norm2"] - 1) < 1e-12
    assert np.abs(x - xo).max() < 1e-10
    psi_o = ohhl.solve(A, b, nc)[2]
    assert abs(rep["p_anc1"] - float(np.sum(np.abs(psi_o[1 << (p.n - 1):]) ** 2))) < 1e-12


def test_table1_on_gpu():
    """PAPER.md:294-296 Table 1 14-bus error 1.97e-3 reproduced by the GPU path (default n_c = 8)."""
    from workloads import matpower
    A, b = matpower.case14()
    x, rep = pkg.hhl_solve(A, b)
    assert rep["n_total"] == 13
    assert abs(np.linalg.norm(x - np.linalg.solve(A, b)) - 1.97e-3) < 0.005e-3


def test_probabilities_after_relabel():
    """Marginals in LOGICAL order even when swaps permuted the physical layout."""
    n = 10
    gates = synthetic.random_circuit(n, 50, seed=9, kmax=2) + [{"kind": "swap", "targets": [0, 9]},
                                                                {"kind": "swap", "targets": [3, 4]}]
    got, ref, st = run_both(n, gates, None, fusion_kmax=3, tile_qubits=6)
    assert st.qubit_map() != list(range(n))
    assert np.abs(got - ref).max() < 1e-10
    for qs in ([0], [9, 0], [3, 4, 5], list(range(n)), [7, 2, 0, 4]):
        assert np.abs(st.probabilities(qs) - sim.marginal(ref, n, qs)).max() < 1e-13


def test_determinism():
    A, b, nc = configs.get("C3")
    st = pkg.State(15)
    prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc)
    prog.run()
    a = st.read()
    n1 = st.norm2()
    prog.run()
    assert np.array_equal(a, st.read())
    assert st.norm2() == n1


def test_edge_cases():
    st = pkg.State(1)
    H = np.array([[1, 1], [1, -1]], complex) / np.sqrt(2)
    st.apply_fused([{"kind": "dense", "targets": [0], "data": H}])
    assert np.abs(st.read() - [2 ** -0.5, 2 ** -0.5]).max() < 1e-15
    amps, idx, p = st.postselect_slice([0], [1])
    assert idx[0] == 1 and abs(p - 0.5) < 1e-15
    # k = n dense on a 5-qubit state, tiles larger than the state
    g = synthetic.rng(1)
    U = synthetic.haar_unitary(5, g)
    got, ref, _ = run_both(5, [{"kind": "dense", "targets": [4, 2, 0, 1, 3], "data": U}],
                           synthetic.random_state(5, 1), fusion_kmax=0, tile_qubits=12)
    assert np.abs(got - ref).max() < 1e-12
    with pytest.raises(pkg.SVError):
        st.apply_fused([{"kind": "dense", "targets": [1], "data": H}])
    with pytest.raises(pkg.SVError):
        st.read(0, 3)


def test_many_tiles_ragged():
    """n = 22: 2^22 amplitudes over many tiles; a circuit touching low, high and middle bits."""
    n = 22
    gates = synthetic.random_circuit(n, 40, seed=22, kmax=3)
    psi0 = synthetic.random_state(n, 22)
    for mode in (dict(tile_qubits=-1), dict(tile_qubits=12, tile_jit=-1), dict(tile_qubits=12, tile_jit=1)):
        got, ref, _ = run_both(n, gates, psi0, fusion_kmax=4, **mode)
        assert np.abs(got - ref).max() < 1e-10


# --------------------------------------------------------------- full size (S30)
def _tol_frontend(p):
    """Independent eigensolvers differ by ~eps·||A||; the HHL state's sensitivity to phi is ~2 pi N_c.
    |d psi| <~ 2 pi N_c · |d phi| with |d phi| <= 8 eps · phi_max."""
    return max(1e-10, 2 * np.pi * (1 << p.n_c) * 8 * np.finfo(float).eps * float(np.max(np.abs(p.phi))))


@pytest.fixture(scope="module")
def s30_reference():
    """Closed-form (oracle) values for S30: P_succ, x~ and sampled amplitudes (~1-2 min of CPU)."""
    A, b, nc = configs.get("S30")
    p = ohhl.plan(A, b, nc)
    xt, P = cf.postselected(p)
    g = synthetic.rng(30)
    idx = np.unique(np.concatenate([g.integers(0, 1 << p.n, 12), [0, 5, (1 << p.n) - 1, 1 << (p.n - 1)]]))
    return A, b, nc, p, xt, P, idx, cf.sampled_amplitudes(p, idx)


@pytest.mark.slow
@pytest.mark.parametrize("opts", [dict(), dict(qpe_mode=1)])
def test_s30_full_size(s30_reference, opts):
    """configs[3] (30 qubits, 16 GiB state) in the launch configuration bench.py times (product
    front end): sampled amplitudes vs the closed form, post-selected x and P_succ within the derived
    front-end tolerance."""
    A, b, nc, p, xt, P, idx, ref = s30_reference
    st = pkg.State(p.n)
    prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, **opts)
    prog.run()
    x, ps = prog.readout()
    tol = _tol_frontend(p)
    assert abs(ps - P) < max(1e-12, tol)
    assert np.abs(x - p.b_norm * xt[: p.n_orig] / p.lam_min).max() < 10 * tol
    got = np.array([st.read(int(i), 1)[0] for i in idx])
    assert np.abs(got - ref).max() < tol
    assert abs(st.norm2() - 1.0) < 1e-11


@pytest.mark.slow
def test_s30_engine_parity_oracle_gates(s30_reference):
    """The engine at full size held to 1e-10: the ORACLE's own S30 gate list (oracle phases) run
    through the product fusion + tile scheduler + kernels vs the oracle closed form."""
    A, b, nc, p, xt, P, idx, ref = s30_reference
    gates = ohhl.build(p)
    st = pkg.State(p.n)
    prog = pkg.Program.create(st, gates, fusion_kmax=2, tile_qubits=12)
    prog.run()
    got = np.array([st.read(int(i), 1)[0] for i in idx])
    assert np.abs(got - ref).max() < 1e-10
    base = 1 << (p.n - 1)
    sl = st.read(base, 1 << p.n_b)
    assert np.abs(sl - xt).max() < 1e-10
    assert abs(float(np.sum(np.abs(sl) ** 2)) - P) < 1e-12


# ------------------------------------------------ virtual shards (multi-GPU logic)
VMODES = [dict(tile_qubits=-1), dict(tile_qubits=8, tile_jit=-1), dict(tile_qubits=8, tile_jit=1)]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", VMODES)
def test_virtual_shards_random_circuits(world, mode):
    """world > 1 without NCCL: the sharded scheduler (exchanges, rank-resolved controls/diagonals),
    the rank_base paths of every kernel and the pack/unpack exchange, vs the unsharded oracle."""
    n = 12
    for seed in range(2):
        gates = synthetic.random_circuit(n, 80, seed=500 + seed + 10 * world, kmax=3)
        psi0 = synthetic.random_state(n, seed)
        st = pkg.State(n, world=world)
        st.write(psi0)
        st.apply_circuit(gates, fusion_kmax=2, **mode)
        ref = sim.run(gates, n, psi0)
        assert np.abs(st.read() - ref).max() < 1e-10
        for qs in ([n - 1], [0, n - 1, n - 2], list(range(4))):
            assert np.abs(st.probabilities(qs) - sim.marginal(ref, n, qs)).max() < 1e-12
        assert abs(st.norm2() - 1.0) < 1e-12


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("opts", [dict(), dict(qpe_mode=1), dict(tile_qubits=-1), dict(tile_jit=1, tile_qubits=9),
                                  configs.BENCH_OPTS, dict(configs.BENCH_OPTS, tile_qubits=8)])
def test_virtual_shards_hhl(world, opts):
    """Sharded HHL (in-process virtual shards). With the bench options (eigenbasis) the top system
    qubits are global and the circuit needs one multi-qubit exchange (all-to-all) before V.
    """
    A, b, nc = configs.get("C3")
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    st = pkg.State(p.n, world=world)
    prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, **opts)
    prog.run()
    assert np.abs(st.read() - psi_o).max() < 1e-10
    x, ps = prog.readout()
    assert abs(ps - po) < 1e-12 and np.abs(x - xo).max() < 1e-10
    x2, rep = pkg.hhl_solve(A, b, clock_qubits=nc, world=world, **opts)
    assert np.abs(x2 - xo).max() < 1e-10


@pytest.mark.parametrize("opts", [dict(), dict(qpe_mode=1), dict(tile_qubits=-1)])
def test_hermitian_embedding_gpu(opts):
    """Non-symmetric systems through the product front end: full state vs oracle."""
    g = synthetic.rng(3)
    cases = [(np.array([[0.0, 1.0], [3.0, 0.0]]), np.array([0.6, 0.8]), 0),
             (g.standard_normal((4, 4)) + 4 * np.eye(4), g.standard_normal(4), 8)]
    for A, b, nc in cases:
        xo, po, psi_o, p = ohhl.solve(A, b, nc or None)
        st = pkg.State(p.n)
        prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, **opts)
        prog.run()
        assert np.abs(st.read() - psi_o).max() < 1e-10
        x, ps = prog.readout()
        assert abs(ps - po) < 1e-12 and np.abs(x - xo).max() < 1e-10


def test_table1_30bus_on_gpu():
    """PAPER.md:294-296 Table 1 30-bus error 1.18e-3 (16 qubits, default n_c = 10) on the GPU path."""
    from workloads import matpower
    A, b = matpower.case30()
    x, rep = pkg.hhl_solve(A, b)
    assert (rep["n_data"], rep["n_clock"], rep["n_total"]) == (5, 10, 16)
    assert abs(np.linalg.norm(x - np.linalg.solve(A, b)) - 1.18e-3) < 0.005e-3


@pytest.mark.parametrize("kinds", [("controlled", "diagonal"), ("dense", "controlled"), ("dense", "diagonal", "swap")])
@pytest.mark.parametrize("T", [7, 8, 9, 12])
def test_jit_small_tiles_wide_ops(kinds, T):
    """NVRTC tile passes at small tiles with 3-qubit (wide) dense/controlled ops: single-phase passes,
    direct HBM<->register phases, thread/tile-controlled wide ops, kernel-parameter matrices
    (regression: an unrolled form of the wide-op row loop miscomputed T=8 controlled kernels)."""
    n = 12
    for seed in range(6):
        gates = synthetic.random_circuit(n, 40, seed=700 + seed, kinds=kinds, kmax=3)
        psi0 = synthetic.random_state(n, seed)
        got, ref, _ = run_both(n, gates, psi0, fusion_kmax=2, tile_qubits=T, tile_jit=1)
        assert np.abs(got - ref).max() < 1e-10, (seed, np.abs(got - ref).max())


@pytest.mark.parametrize("mode", [dict(tile_qubits=-1), dict(tile_qubits=8, tile_jit=1), dict(tile_qubits=8, tile_jit=-1)])
def test_paper_mode_fusion_transpiled_hhl(mode):
    """Fig. 4 fusion (fusion_mode = 1) on the transpiled 2x2 HHL stream:
    GPU state vs the oracle's unfused run, and the HHL post-selection of the 5-qubit register."""
    from oracle import transpile as tr
    A, b, nc = configs.get("C1")
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    t = tr.transpile(p.gates)
    for n in (p.n, 10):
        got, ref, st = run_both(n, t, None, fusion_mode=1, **mode)
        assert np.abs(got - ref).max() < 1e-10
    got5, _, _ = run_both(p.n, t, None, fusion_mode=1, **mode)
    assert np.abs(got5 - psi_o).max() < 1e-10


@pytest.mark.parametrize("n,sampled", [(22, False), (30, True)])
def test_padded_stress_circuit_tensor_factor(n, sampled):
    """SURVEY §8(d) padded stress circuits P_n: C3's 15-qubit textbook HHL list on a seeded random
    injective qubit map + brickwork pad layers. Tensor-factor pin: psi = perm(psi_HHL15 (x) psi_pad),
    both factors from the small oracle runs. P22: every amplitude; P30 (16 GiB): 256 random
    amplitudes plus the HHL factor's post-selection slice (pad factor at its first basis state)."""
    A, b, nc = configs.get("C3")
    p = ohhl.plan(A, b, nc)
    g15 = ohhl.build(p)
    gates, qmap, pad = synthetic.padded_circuit(g15, p.n, n)
    psi15 = sim.run(g15, p.n)
    psipad = sim.run(synthetic.pad_brickwork(list(range(n - p.n))), n - p.n)
    st = pkg.State(n)
    prog = pkg.Program.create(st, gates, fusion_kmax=2, tile_qubits=12)
    prog.run()
    if not sampled:
        idx = np.arange(1 << n)
        got = st.read()
    else:
        g = synthetic.rng(n)
        idx = np.unique(g.integers(0, 1 << n, 1 << 17))
        got = np.concatenate([st.read(int(i), 1) for i in idx[:256]])
        idx = idx[:256]
        # the HHL factor's post-selected slice with the pad factor at its first basis state
        base = 1 << (p.n - 1)
        sl = np.arange(base, base + (1 << p.n_b))
        full_sl = np.zeros(sl.size, dtype=np.int64)
        for j, q in enumerate(qmap):
            full_sl |= ((sl >> j) & 1) << q
        idx = np.concatenate([idx, full_sl])
        got = np.concatenate([got, [st.read(int(i), 1)[0] for i in full_sl]])
    ref = synthetic.tensor_factor_amplitudes(psi15, qmap, psipad, pad, idx)
    err = float(np.abs(got - ref).max())
    print(f"\n[parity] P{n} padded stress circuit ({len(gates)} gates): max|psi - tensor factors| = {err:.3e}")
    assert err < 1e-10


def test_dump_restore_checkpoint(tmp_path):
    """sv_dump / sv_restore (SPEC "External Interfaces"): uint64 length header + interleaved re/im
    doubles, little-endian, logical order -- read back by numpy -- and a restore into another state
    (after a permuting circuit, so logical != physical order)."""
    n = 12
    gates = synthetic.random_circuit(n, 30, seed=4, kmax=2) + [{"kind": "swap", "targets": [0, 11]}]
    got, ref, st = run_both(n, gates, synthetic.random_state(n, 4), fusion_kmax=2, tile_qubits=8)
    path = str(tmp_path / "state.bin")
    st.dump(path)
    raw = np.fromfile(path, dtype="<u8", count=1)
    assert int(raw[0]) == 1 << n
    data = np.fromfile(path, dtype="<f8", offset=8).view(np.complex128)
    assert np.array_equal(data, got)
    st2 = pkg.State(n)
    st2.restore(path)
    assert np.array_equal(st2.read(), got)
    st3 = pkg.State(n + 1)
    with pytest.raises(pkg.SVError):
        st3.restore(path)


def test_random_hermitian_systems():
    """SPEC acceptance 5 as test idea: 50 seeded random symmetric systems (dim 2 and 4, kappa <= 8,
    some negative eigenvalues) through hhl_solve: x equal to the oracle's HHL x (1e-10) at n_qpe = 8 --
    the parity bar. Accuracy vs the dense direct solve is a property of HHL at this clock size, not of the
    simulator: with the paper's qlsarepo conventions (R4) the median relative error is 1e-2 and 86 % are
    below SPEC's 5e-2 (checked here as median < 2e-2, max < 0.25). Systems with exactly representable
    eigenvalues: 1e-8."""
    g = synthetic.rng(611)
    rel = []
    for i in range(50):
        d = 2 if i % 2 == 0 else 4
        Q, _ = np.linalg.qr(g.standard_normal((d, d)))
        lam = g.uniform(1.0, 8.0, d) * np.where(g.random(d) < 0.3, -1.0, 1.0)
        lam[0] = 1.0 if abs(lam[0]) < 1 else lam[0]
        if np.abs(lam).max() / np.abs(lam).min() > 8:
            lam = np.sign(lam) * np.clip(np.abs(lam), 1.0, 8.0)
        A = (Q * lam) @ Q.T
        A = (A + A.T) / 2
        b = g.standard_normal(d)
        x, rep = pkg.hhl_solve(A, b, clock_qubits=8)
        xo, po, _, p = ohhl.solve(A, b, 8)
        assert np.abs(x - xo).max() < 1e-10
        xt = np.linalg.solve(A, b)
        rel.append(np.linalg.norm(x - xt) / np.linalg.norm(xt))
    assert np.median(rel) < 2e-2 and max(rel) < 0.25
    for lam in ([1.0, 2.0], [1.0, 4.0], [0.5, 1.0, 2.0, 4.0]):
        d = len(lam)
        Q, _ = np.linalg.qr(g.standard_normal((d, d)))
        A = (Q * np.array(lam)) @ Q.T
        A = (A + A.T) / 2
        b = g.standard_normal(d)
        x, rep = pkg.hhl_solve(A, b, clock_qubits=6)
        xt = np.linalg.solve(A, b)
        assert np.linalg.norm(x - xt) / np.linalg.norm(xt) < 1e-8, lam


@pytest.mark.parametrize("nc", [3, 4, 5])
def test_qpe_exact_on_gpu(nc):
    """SPEC acceptance 6: QPE on an eigenvector with a representable eigenphase puts probability
    >= 1 - 1e-9 on the correct clock bitstring (GPU run of the oracle's H / c-U / IQFT list)."""
    A = np.diag([1.0, 3.0])
    p = ohhl.plan(A, np.ones(2), nc)
    gates = ohhl.build(p)
    q = gates[1: 1 + 2 * nc + nc + nc * (nc - 1) // 2 + nc // 2]
    for s in range(2):
        psi0 = np.zeros(1 << p.n, complex)
        psi0[: 1 << p.n_b] = p.V[:, s]
        st = pkg.State(p.n)
        st.write(psi0)
        st.apply_circuit(q, fusion_kmax=2)
        probs = st.probabilities(list(range(p.n_b, p.n_b + nc)))
        m0 = round(p.phi[s] * (1 << nc))
        assert probs[m0] >= 1 - 1e-9
