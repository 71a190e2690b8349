"""Shot sampling (SPEC `sample` S:166-174; Fig. 3 caption: "10,000 measurements of bell
state"): oracle pins (CPU) and the library's sv_sample vs the oracle, index for index (GPU)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import sample as osample
from workloads import synthetic


def test_zero_state_all_zero_index():
    psi = np.zeros(8, dtype=complex)
    psi[0] = 1.0
    assert (osample.sample(psi, 100, seed=1) == 0).all()


def test_bell_counts_fig3():
    """Fig. 3: only 00 and 11 appear; each within 5 sigma of 5000 in 10,000 shots."""
    psi = np.zeros(4, dtype=complex)
    psi[0] = psi[3] = 1 / np.sqrt(2)
    s = osample.sample(psi, 10000, seed=2402)
    c = np.bincount(s.astype(np.int64), minlength=4)
    assert c[1] == 0 and c[2] == 0
    assert abs(c[0] - 5000) < 5 * 50 and c[0] + c[3] == 10000


def test_deterministic_in_seed():
    psi = synthetic.random_state(6, 3)
    a, b = osample.sample(psi, 500, seed=11), osample.sample(psi, 500, seed=11)
    c = osample.sample(psi, 500, seed=12)
    assert (a == b).all() and not (a == c).all()


def test_uniform_generator_splitmix64_reference():
    # splitmix64 reference output for state 0 after one increment (Vigna's published first value)
    assert osample.splitmix64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    u = osample.uniforms(7, 1000)
    assert (u >= 0).all() and (u < 1).all() and abs(u.mean() - 0.5) < 0.05


@pytest.mark.parametrize("n", [3, 8, 10])
def test_matches_plain_inverse_cdf(n):
    """Single block (n <= 10): the fixed-order procedure equals textbook inverse-CDF sampling
    (sequential cumulative sum + first index above u * total)."""
    psi = synthetic.random_state(n, n)
    u = osample.uniforms(5, 2000)
    p = np.abs(psi) ** 2
    cdf = np.cumsum(p)
    plain = np.searchsorted(cdf, u * cdf[-1], side="right")
    assert (osample.sample(psi, 2000, seed=5) == plain).all()


def test_chi_square_random_state():
    n = 4
    psi = synthetic.random_state(n, 9)
    shots = 40000
    c = np.bincount(osample.sample(psi, shots, seed=9).astype(np.int64), minlength=16)
    e = shots * np.abs(psi) ** 2
    chi2 = ((c - e) ** 2 / e).sum()
    assert chi2 < 45.0            # 15 dof: P(chi2 > 45) ~ 1e-4


def test_multi_level_consistent_with_block_cdf():
    """n = 22 (4 superblocks of 1024 blocks): every sample's index lies where the plain CDF puts
    its uniform up to the rounding of the summation order (the chosen index's CDF interval, widened by
    1e-12, contains u * total)."""
    n = 22
    psi = synthetic.random_state(n, 4)
    s = osample.sample(psi, 300, seed=4).astype(np.int64)
    p = np.abs(psi) ** 2
    cdf = np.cumsum(p)
    t = osample.uniforms(4, 300) * cdf[-1]
    lo = np.where(s > 0, cdf[np.maximum(s - 1, 0)], 0.0)
    assert ((lo - 1e-12 <= t) & (t < cdf[s] + 1e-12)).all()


@pytest.mark.parametrize("n", [12, 21, 22])
def test_multi_level_equals_plain_inverse_cdf_dyadic(n):
    """Several blocks / superblocks (n > 10): on a state whose probabilities are dyadic with few
    significant bits (a_i = d_i 2^-8, d_i in -3..3) every partial sum is exact in fp64 whatever the
    summation order, so the multi-level procedure must equal textbook inverse-CDF sampling index for
    index (ties cannot be broken differently: all CDF values are exact)."""
    g = synthetic.rng(1000 + n)
    d = g.integers(-3, 4, size=(1 << n, 2)).astype(np.float64)
    d[g.random(1 << n) < 0.3] = 0.0                      # zero runs: empty blocks/elements are skipped
    psi = (d[:, 0] + 1j * d[:, 1]) * 2.0 ** -8
    shots = 3000
    p = psi.real * psi.real + psi.imag * psi.imag
    cdf = np.cumsum(p)
    plain = np.searchsorted(cdf, osample.uniforms(11, shots) * cdf[-1], side="right")
    assert (osample.sample(psi, shots, seed=11) == plain).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n,shots", [(3, 1000), (12, 5000), (22, 2000)])
def test_gpu_sample_matches_oracle(n, shots):
    import paper_2402_08136_b200 as pkg
    psi = synthetic.random_state(n, n + 1)
    st = pkg.State(n)
    st.write(psi)
    got = st.sample(shots, seed=2402 + n)
    ref = osample.sample(st.read(), shots, seed=2402 + n)
    assert (got == ref).all(), np.nonzero(got != ref)[0][:10]


@pytest.mark.gpu
def test_gpu_sample_permuted_map_and_errors():
    """After swaps the library's physical layout differs from the logical order: samples are still
    LOGICAL indices, identical to the oracle's on the logical state."""
    import paper_2402_08136_b200 as pkg
    n = 14
    gates = synthetic.random_circuit(n, 60, seed=31, kmax=2) + [{"kind": "swap", "targets": [0, n - 1]},
                                                                 {"kind": "swap", "targets": [1, 7]}]
    st = pkg.State(n)
    st.write(synthetic.random_state(n, 31))
    st.apply_circuit(gates, fusion_kmax=2)
    assert list(st.qubit_map()) != list(range(n))
    got = st.sample(3000, seed=99)
    assert (got == osample.sample(st.read(), 3000, seed=99)).all()
    st.write(np.zeros(1 << n, dtype=complex))
    with pytest.raises(pkg.SVError):
        st.sample(10, seed=1)


@pytest.mark.gpu
def test_gpu_sample_sharded_state_refused():
    """sv_sample is single-rank (DESIGN.md §6 Sampling): a sharded state reports SV_E_ARG, no fallback."""
    import paper_2402_08136_b200 as pkg
    st = pkg.State(10, world=2)
    st.write(synthetic.random_state(10, 1))
    with pytest.raises(pkg.SVError):
        st.sample(10, seed=1)


@pytest.mark.gpu
def test_gpu_sample_s30_postselection_rate():
    """Full bench size (S30, 2^30 amplitudes, the bench's launch configuration): 10^5 shots from the
    final HHL state; the fraction with ancilla = 1 and clock = 0 (R7) matches P_succ
    within 5 sigma, and every post-selected shot's system index lies in the 16-state data register."""
    import paper_2402_08136_b200 as pkg
    from workloads import configs
    A, b, nc = configs.get("S30")
    n = configs.n_qubits("S30")
    st = pkg.State(n)
    prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, fusion_kmax=1, tile_qubits=12, qpe_mode=1)
    prog.run()
    _, p_succ = prog.readout()
    shots = 100000
    s = st.sample(shots, seed=2402).astype(np.uint64)
    anc = (s >> np.uint64(n - 1)) & np.uint64(1)
    clock = (s >> np.uint64(4)) & np.uint64((1 << nc) - 1)
    hit = (anc == 1) & (clock == 0)
    frac = hit.mean()
    sigma = np.sqrt(p_succ * (1 - p_succ) / shots)
    assert abs(frac - p_succ) < 5 * sigma, (frac, p_succ)
    # the post-selected shots are the slice's logical indices: 2^(n-1) + s_sys, s_sys < 16
    assert ((s[hit] - np.uint64(1 << (n - 1))) < np.uint64(16)).all()
