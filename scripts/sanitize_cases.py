"""Small GPU workload for compute-sanitizer (memcheck / racecheck / synccheck), VERDICT r01 item 3.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
Runs, through the C ABI, the NVRTC tile kernels at T = 7..12 with wide (3-qubit) dense / controlled /
diagonal ops (the shapes of tests/test_gpu_parity.py::test_jit_small_tiles_wide_ops), the C1-C3 HHL
programs with the bench options and the default options, and one forced-JIT 20-qubit HHL-shaped program
(S16..S20 configs), checking each result against the oracle so a silent race also fails here.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402
from oracle import hhl as ohhl  # noqa: E402
from oracle import sim  # noqa: E402
from workloads import configs, synthetic  # noqa: E402

worst = 0.0
n = 12
for kinds in [("controlled", "diagonal"), ("dense", "controlled"), ("dense", "diagonal", "swap")]:
    for T in (7, 8, 9, 12):
        for seed in range(2):
            gates = synthetic.random_circuit(n, 40, seed=700 + seed, kinds=kinds, kmax=3)
            psi0 = synthetic.random_state(n, seed)
            st = pkg.State(n)
            st.write(psi0)
            st.apply_circuit(gates, fusion_kmax=2, tile_qubits=T, tile_jit=1)
            worst = max(worst, float(np.abs(st.read() - sim.run(gates, n, psi0)).max()))
            st.destroy()
for name in ("C1", "C2", "C3", "S18"):
    A, b, nc = configs.get(name)
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    for opts in (configs.BENCH_OPTS, dict(tile_jit=1, tile_qubits=9), dict()):
        st = pkg.State(p.n)
        prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, **opts)
        prog.run()
        worst = max(worst, float(np.abs(st.read() - psi_o).max()))
        prog.readout()
        prog.destroy()
        st.destroy()
print(f"sanitize cases done: max |psi - oracle| = {worst:.3e}")
sys.exit(0 if worst < 1e-10 else 1)
