"""debug: virtual-shard random circuits vs oracle (GPU)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_08136_b200 as pkg
from oracle import sim
from workloads import synthetic
n = 12
for world in (1, 2):
    for T in (8, 9):
        for seed in range(2):
            gates = synthetic.random_circuit(n, 80, seed=500 + seed + 10 * 2, kmax=3)
            psi0 = synthetic.random_state(n, seed)
            st = pkg.State(n, world=world)
            st.write(psi0)
            st.apply_circuit(gates, fusion_kmax=2, tile_qubits=T, tile_jit=1)
            ref = sim.run(gates, n, psi0)
            print(world, T, seed, np.abs(st.read() - ref).max(), flush=True)
