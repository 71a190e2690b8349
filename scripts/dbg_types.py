"""debug: which gate kinds break the JIT tile path at small T (GPU)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_08136_b200 as pkg
from oracle import sim
from workloads import synthetic
n = 12
for kinds in (("dense",), ("controlled",), ("dense", "diagonal"), ("controlled", "diagonal"), ("dense", "swap"), ("dense", "controlled")):
    for kmax in (2, 3):
        for T in (8, 9):
            bad = 0
            for seed in range(6):
                gates = synthetic.random_circuit(n, 40, seed=700 + seed, kinds=kinds, kmax=kmax)
                psi0 = synthetic.random_state(n, seed)
                st = pkg.State(n)
                st.write(psi0)
                st.apply_circuit(gates, fusion_kmax=2, tile_qubits=T, tile_jit=1)
                ref = sim.run(gates, n, psi0)
                bad += np.abs(st.read() - ref).max() > 1e-10
            print(kinds, kmax, T, "bad", bad, "/ 6", flush=True)
