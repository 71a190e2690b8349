"""Named HHL workloads (BASELINE.json ``configs``).

Each config is (A, b, clock_qubits) with A the UNPADDED real-symmetric system
matrix and b the unnormalised right-hand side. Padding, normalisation and the
whole HHL construction are method arithmetic and are done independently by the
oracle and by the product.

    C1   3-bus triangle          2×2    n_c = 3    5 qubits   (configs[0])
    C2   PJM case5, slack 4      4×4    n_c = 6    9 qubits   (configs[1])
    C3   IEEE case14, slack 1   13→16   n_c = 10  15 qubits   (configs[2])
    C3p  IEEE case14 at Table 1's n_QPE = 8                13 qubits
    S16..S29  case14 system, n_c = 11..24 (parity cases between C3 and S30)
    S30  case14 system, n_c = 25                           30 qubits (configs[3])
    S31..S34  n_c = 26..29                                 31..34 qubits (configs[4])
    B30  IEEE case30        29→32  n_c = 10  16 qubits   (Table 1 column 2; NEXT f3)
"""
from __future__ import annotations

from . import matpower

CONFIGS = {
    "C1": (matpower.three_bus, 3),
    "C2": (matpower.case5, 6),
    "C3": (matpower.case14, 10),
    "C3p": (matpower.case14, 8),
    "B30": (matpower.case30, 10),
}
for _n in range(16, 35):
    CONFIGS[f"S{_n}"] = (matpower.case14, _n - 5)


def get(name: str):
    """Return (A, b, clock_qubits) for a named config."""
    fn, nc = CONFIGS[name]
    A, b = fn()
    return A, b, nc


def n_qubits(name: str) -> int:
    """Total qubits n = n_b + n_c + 1 with n_b = ceil(log2(rows))."""
    A, _, nc = get(name)
    nb = max(1, (A.shape[0] - 1).bit_length())
    return nb + nc + 1


# The launch configuration bench.py times (its argparse defaults): fusion k_max 1, 12-qubit tile
# passes, eigenbasis QPE, NVRTC-specialised tile passes forced on (the bench's 2^30
# amplitudes would pick them anyway; forcing them makes small parity cases run the same generator).
BENCH_OPTS = dict(fusion_kmax=1, tile_qubits=12, qpe_mode=1, tile_jit=1)


def describe(name: str) -> str:
    """One-line description of a config's linear system (for bench lines)."""
    fn, nc = CONFIGS[name]
    A, _ = fn()
    src = {"three_bus": "3-bus triangle DC B", "case5": "PJM 5-bus DC B (MATPOWER case5)",
           "case14": "IEEE 14-bus DC B (MATPOWER case14)", "case30": "IEEE 30-bus DC B (MATPOWER case30)"}
    N0 = A.shape[0]
    Np = 1 << max(1, (N0 - 1).bit_length())
    return f"{src.get(fn.__name__, fn.__name__)}, {N0}x{N0} -> {Np}x{Np}, n_c = {nc}"
