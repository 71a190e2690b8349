"""One tile pass of K Hadamards on high qubits (developer microbenchmark for ncu)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402

n = int(os.environ.get("N", "30"))
K = int(os.environ.get("K", "7"))
T = int(os.environ.get("T", "12"))
H = np.array([[1, 1], [1, -1]], complex) / np.sqrt(2)
st = pkg.State(n)
gates = [{"kind": "dense", "targets": [n - 1 - i], "data": H} for i in range(K)]
prog = pkg.Program.create(st, gates, fusion_kmax=1, tile_qubits=T)
prog.set_timing(True)
for _ in range(3):
    prog.run()
    t = prog.timings()
print(prog.dump())
print(f"K={K} T={T}: {t[0][0]:.3f} ms  {32 * 2**n / t[0][0] / 1e6:.0f} GB/s")
