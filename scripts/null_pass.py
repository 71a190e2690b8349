"""Tile-kernel streaming floor: a 30-qubit program of k one-qubit gates on high qubits (one register
phase, direct HBM in/out) timed per pass (developer tool, GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_08136_b200 as pkg
n = 30
H = np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2)
st = pkg.State(n)
for qs in ([24], [24, 25, 26, 27], list(range(20, 28))):
    gates = [{"kind": "dense", "targets": [q], "data": H} for q in qs]
    prog = pkg.Program.create(st, gates, fusion_kmax=1, tile_qubits=12, tile_jit=1)
    prog.set_timing(True)
    for _ in range(4):
        prog.run()
    t = prog.timings()
    print(len(qs), "H gates:", [f"{x[0]:.3f} ms" for x in t], prog.dump().splitlines()[0][:80], flush=True)
    prog.destroy()
