"""Micro-variants of the eigenbasis 'D^dagger + V' tile pass (developer tool)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402

n = 30
g = np.random.default_rng(0)
H = np.array([[1, 1], [1, -1]], complex) / np.sqrt(2)
V = np.linalg.qr(g.standard_normal((16, 16)))[0].astype(complex)
D = [{"kind": "diagonal", "targets": [0, 1, 2, 3] + [4 + 4 * c + i for i in range(4) if 4 + 4 * c + i < 29],
      "data": None} for c in range(7)]
for d in D:
    d["data"] = np.exp(2j * np.pi * g.random(1 << len(d["targets"])))
Vg = [{"kind": "dense", "targets": [0, 1, 2, 3], "data": V}]
Hs = [{"kind": "dense", "targets": [q], "data": H} for q in (5, 6, 7, 8, 9, 28)]
st = pkg.State(n)
for name, gates in [("D+V+H", D + Vg + Hs), ("D+H", D + Hs), ("V+H", Vg + Hs), ("H", Hs), ("D", D), ("V", Vg)]:
    for T in (10, 11):
        prog = pkg.Program.create(st, gates, fusion_kmax=1, tile_qubits=T, tile_jit=1)
        prog.set_timing(True)
        for _ in range(3):
            prog.run()
            t = prog.timings()
        print(f"{name:8s} T={T}: " + " ".join(f"{x[0]:.2f}" for x in t) + f"  total {sum(x[0] for x in t):.2f} ms")
        prog.destroy()
