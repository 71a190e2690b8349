"""Developer check (GPU): the transpiled 2x2 HHL stream with Fig. 4 fusion at T = 8 (JIT) vs the oracle,
under the JIT configuration given in HHLSV_JIT (e.g. ptxas=-O1, clobber=1)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402
from oracle import hhl as ohhl, sim, transpile as tr  # noqa: E402
from workloads import configs, synthetic  # noqa: E402
A, b, nc = configs.get("C1")
p = ohhl.plan(A, b, nc)
t = tr.transpile(ohhl.build(p))
for n, T, seed in [(10, 8, None), (10, 8, 3), (10, 9, None), (12, 8, None)]:
    psi0 = None if seed is None else synthetic.random_state(n, seed)
    st = pkg.State(n)
    if psi0 is not None:
        st.write(psi0)
    st.apply_circuit(t, fusion_mode=1, tile_qubits=T, tile_jit=1)
    err = np.abs(st.read() - sim.run(t, n, psi0)).max()
    print(f"HHLSV_JIT={os.environ.get('HHLSV_JIT', '')!r} n={n} T={T} psi0={'zero' if seed is None else seed}: max err {err:.3e}")
