"""One k = 5 dense op on a 2^n state through the streaming path (the DMMA kernel), for ncu (developer tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
rng = np.random.default_rng(7)
U = np.linalg.qr(rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32)))[0]
st = pkg.State(n)
for t in ([0, 1, 2, 3, 4], [n - 5, n - 4, n - 3, n - 2, n - 1]):
    prog = pkg.Program.create(st, [{"kind": "dense", "targets": t, "data": U}], fusion_kmax=5, tile_qubits=-1, tile_jit=-1)
    for _ in range(3):
        prog.run()
    prog.destroy()
st.sync() if hasattr(st, "sync") else None
print("ok")
