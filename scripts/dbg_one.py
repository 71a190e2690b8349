"""debug: one random circuit (n=12, T=8, JIT) vs the oracle (GPU)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_08136_b200 as pkg
from oracle import sim
from workloads import synthetic
n = 12
gates = synthetic.random_circuit(n, 80, seed=int(os.environ.get("SEED", "520")), kmax=3, **({"kinds": ("controlled", "diagonal")} if os.environ.get("CD") else {}))
psi0 = synthetic.random_state(n, 0)
st = pkg.State(n)
st.write(psi0)
st.apply_circuit(gates, fusion_kmax=2, tile_qubits=int(os.environ.get("T", "8")), tile_jit=1)
ref = sim.run(gates, n, psi0)
print("err", np.abs(st.read() - ref).max(), flush=True)
if os.environ.get("HHLSV_EMU_DUMP"):
    d = os.environ["HHLSV_EMU_DUMP"]
    np.save(os.path.join(d, "psi0.npy"), psi0)
    np.save(os.path.join(d, "gpu.npy"), st.read())
    np.save(os.path.join(d, "ref.npy"), ref)
