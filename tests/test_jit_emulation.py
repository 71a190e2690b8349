"""CPU checks of the GENERATED tile kernels (no GPU): host emulation with race / bounds / barrier
checking (tests/jit_emulator.py), standing in for compute-sanitizer, which is closed on the GPU pool.

The library's host-only planner exports each program exactly as it would run on the B200 (same
scheduler, lowering and CUDA source generator); the emulator runs every pass thread by thread and the
final state is compared with the oracle. Uninitialised device memory is modelled by NaN: a pass that
read an amplitude the schedule treats as known-zero (lazy qubits) or a stale shared-memory word
would poison the result.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2402_08136_b200 as pkg
from oracle import hhl as ohhl
from oracle import sim
from workloads import configs, synthetic

import jit_emulator as emu


def _export(tmp_path, fn):
    d = str(tmp_path)
    old = os.environ.get("HHLSV_EMU_DIR")
    os.environ["HHLSV_EMU_DIR"] = d
    try:
        txt = fn()
    finally:
        if old is None:
            os.environ.pop("HHLSV_EMU_DIR", None)
        else:
            os.environ["HHLSV_EMU_DIR"] = old
    return d, txt


def _clean(reports):
    for r in reports:
        assert r["races"] == 0 and r["oob"] == 0 and r["double_writes"] == 0 and r["sync_mismatch"] == 0, r


def test_bench_program_c3_emulated(tmp_path):
    """The bench options on C3 (15 qubits): fused product init, lazy ancilla (pass 1 skips its tiles,
    pass 2 reads only its zero half), constant-bank tables, direct HBM phases; from NaN memory."""
    A, b, nc = configs.get("C3")
    d, txt = _export(tmp_path, lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, fused_marginal=1,
                                                             **configs.BENCH_OPTS)[0])
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    out, reps = emu.run_program(d, np.full(1 << p.n, np.nan + 1j * np.nan))
    _clean(reps)
    assert len(reps) >= 2
    assert np.abs(emu.to_logical(out, emu.final_map(txt)) - psi_o).max() < 1e-12
    # fused marginal of the last pass: P(ancilla = 0 / 1) accumulated while it stores the final state
    # (the ancilla is logical qubit n-1: the upper half of the logical index space)
    h = 1 << (p.n - 1)
    want = (np.sum(np.abs(psi_o[:h]) ** 2), np.sum(np.abs(psi_o[h:]) ** 2))
    assert "red" in reps[-1] and all("red" not in r for r in reps[:-1])
    assert np.allclose(reps[-1]["red"], want, rtol=0, atol=1e-13), (reps[-1]["red"], want)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_single_tile_programs_emulated(tmp_path, name):
    """Table 1 regime: a state no larger than one tile (C1: 5 qubits -> T = 5, 2 threads; C2: 9 qubits)
    runs the whole HHL circuit as ONE generated pass (one launch)."""
    A, b, nc = configs.get(name)
    d, txt = _export(tmp_path, lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, **configs.BENCH_OPTS)[0])
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    out, reps = emu.run_program(d, np.full(1 << p.n, np.nan + 1j * np.nan))
    _clean(reps)
    assert len(reps) == 1
    assert np.abs(emu.to_logical(out, emu.final_map(txt)) - psi_o).max() < 1e-12


def test_small_tile_wide_ops_emulated(tmp_path):
    """Random circuit with 3-qubit controlled / diagonal ops at T = 8 (the shapes whose variants gave
    wrong GPU amplitudes in round 1): single-phase passes, controls on thread bits, kernel-parameter
    matrices, cp.async loads; several persistent CTAs with more than one tile each."""
    n = 12
    gates = synthetic.random_circuit(n, 40, seed=703, kinds=("controlled", "diagonal"), kmax=3)
    psi0 = synthetic.random_state(n, 3)
    d, txt = _export(tmp_path, lambda: pkg.schedule_dump(n, gates, fusion_kmax=2, tile_qubits=8, tile_jit=1)[0])
    out, reps = emu.run_program(d, psi0)
    _clean(reps)
    ref = sim.run(gates, n, psi0)
    assert np.abs(emu.to_logical(out, emu.final_map(txt)) - ref).max() < 1e-12


def test_race_detector_catches_a_missing_barrier(tmp_path):
    """Negative control: the same C3 pass with one phase barrier deleted must be reported as racy."""
    A, b, nc = configs.get("C3")
    d, _ = _export(tmp_path, lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, **configs.BENCH_OPTS)[0])
    with open(os.path.join(d, "launches.txt")) as f:
        tiles = [ln.split() for ln in f if ln.startswith("TILE")]
    t = tiles[-1]
    src_path = os.path.join(d, f"src_{t[1]}.cu")
    with open(src_path) as f:
        src = f.read()
    k = src.index("      bar();\n    }\n")             # the barrier closing the first register phase
    with open(src_path, "w") as f:
        f.write(src[:k] + src[k + len("      bar();\n"):])
    with open(os.path.join(d, "launches.txt"), "w") as f:
        f.write(" ".join(t) + "\n")
    _, reps = emu.run_program(d, synthetic.random_state(15, 1))
    assert reps[0]["races"] > 0


def test_paper_mode_fusion_emulated(tmp_path):
    """Fig. 4 fusion (fusion_mode = 1) of the transpiled 2x2 HHL stream, placed on a 10-qubit register so
    the program runs as tile passes: emulated kernels vs the oracle's run of the unfused stream."""
    from oracle import transpile as tr
    A, b, nc = configs.get("C1")
    p = ohhl.plan(A, b, nc)
    t = tr.transpile(ohhl.build(p))
    n = 10
    psi0 = synthetic.random_state(n, 11)
    d, txt = _export(tmp_path, lambda: pkg.schedule_dump(n, t, fusion_mode=1, tile_qubits=8, tile_jit=1)[0])
    out, reps = emu.run_program(d, psi0)
    _clean(reps)
    assert np.abs(emu.to_logical(out, emu.final_map(txt)) - sim.run(t, n, psi0)).max() < 1e-12


@pytest.mark.parametrize("ctrls", ["d,d,11", "12,11,10", "d,11,12,10,13"])
def test_wide_run_products_emulated(tmp_path, ctrls):
    """Per-tile products of a run of 4-qubit dense / controlled ops on the phase's register bits (controls
    out of the tile and on <= 2 thread bits): the CTA multiplies the matrices per thread-bit combination
    and every thread applies one product."""
    n = 15
    rng = np.random.default_rng(5)

    def unitary():
        z = rng.normal(size=(16, 16)) + 1j * rng.normal(size=(16, 16))
        return np.linalg.qr(z)[0]
    gates = []
    for c in ctrls.split(","):
        if c == "d":
            gates.append({"kind": "dense", "targets": [0, 1, 2, 3], "data": unitary()})
        else:
            gates.append({"kind": "controlled", "targets": [0, 1, 2, 3], "controls": [int(c)], "cvals": 1,
                          "data": unitary()})
    psi0 = synthetic.random_state(n, 2)
    d, txt = _export(tmp_path, lambda: pkg.schedule_dump(n, gates, fusion_kmax=1, tile_qubits=12, tile_jit=1)[0])
    srcs = [open(os.path.join(d, f)).read() for f in os.listdir(d) if f.startswith("src_")]
    assert sum(s.count("wide run") for s in srcs) == 1
    out, reps = emu.run_program(d, psi0)
    _clean(reps)
    assert np.abs(emu.to_logical(out, emu.final_map(txt)) - sim.run(gates, n, psi0)).max() < 1e-12


def test_textbook_hhl_wide_run_emulated(tmp_path):
    """C3's textbook circuit (controlled-U^(2^j) chain on the system register) as 12-qubit tile passes:
    the chain runs as per-tile products; the state matches the oracle."""
    A, b, nc = configs.get("C3")
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    d, txt = _export(tmp_path, lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, tile_jit=1, tile_qubits=12,
                                                             fusion_kmax=4, qpe_mode=0)[0])
    srcs = [open(os.path.join(d, f)).read() for f in os.listdir(d) if f.startswith("src_")]
    assert sum(s.count("wide run") for s in srcs) >= 1
    out, reps = emu.run_program(d, np.full(1 << p.n, np.nan + 1j * np.nan))
    _clean(reps)
    assert np.abs(emu.to_logical(out, emu.final_map(txt)) - psi_o).max() < 1e-12
