"""debug: (controlled, diagonal) kmax 3 circuits at T=8 per seed (GPU)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_08136_b200 as pkg
from oracle import sim
from workloads import synthetic
n = 12
for seed in [int(x) for x in os.environ.get("SEEDS", "700 701 702 703 704 705").split()]:
    gates = synthetic.random_circuit(n, 40, seed=seed, kinds=("controlled", "diagonal"), kmax=3)
    psi0 = synthetic.random_state(n, seed - 700)
    st = pkg.State(n)
    st.write(psi0)
    st.apply_circuit(gates, fusion_kmax=2, tile_qubits=int(os.environ.get("T", "8")), tile_jit=1)
    ref = sim.run(gates, n, psi0)
    print(seed, np.abs(st.read() - ref).max(), flush=True)
