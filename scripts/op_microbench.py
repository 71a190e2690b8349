"""Single fused-op kernel GB/s (SURVEY §8(d) "micro" config; developer tool, GPU).

A random complex-Gaussian 2^n state (seed 7); one fused op per kind x k x target placement, run as ONE
streaming pass (tile_qubits = -1: the a4-a6 kernels k_dense / k_diag) and as one generated tile pass
(tile_qubits = 12, NVRTC), timed with CUDA events (median of 5 launches). Bytes = the op's own HBM
traffic (32 B per amplitude it touches: controls select 2^-c of the state). One JSON line per case.

    python scripts/op_microbench.py [n=30] > profiles/r02_op_microbench.jsonl
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
rng = np.random.default_rng(7)
st = pkg.State(n)
chunk = 1 << 24
for first in range(0, 1 << n, chunk):          # seeded complex-Gaussian state, written in chunks
    z = rng.normal(size=chunk) + 1j * rng.normal(size=chunk)
    st.write(z / np.sqrt(2.0 * (1 << n)), first)


def placements(k):
    return {"low": list(range(k)), "mid": [n // 2 + i for i in range(k)], "top": [n - 1 - i for i in range(k)],
            "split": [i for i in range((k + 1) // 2)] + [n - 1 - i for i in range(k // 2)]}


def unitary(k):
    z = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
    return np.linalg.qr(z)[0]


for kind in ("dense", "controlled", "diagonal"):
    for k in range(1, 6):
        for place, t in placements(k).items():
            if kind == "controlled":
                ctrl = [n // 2 - 1]                      # one control between the blocks
                if ctrl[0] in t:
                    continue
                g = {"kind": "controlled", "targets": t, "controls": ctrl, "cvals": 1, "data": unitary(k)}
                frac = 0.5
            elif kind == "dense":
                g, frac = {"kind": "dense", "targets": t, "data": unitary(k)}, 1.0
            else:
                g, frac = {"kind": "diagonal", "targets": t, "data": np.exp(1j * rng.uniform(0, 6, 1 << k))}, 1.0
            for mode, tq in (("streaming", -1), ("tile", 12)):
                prog = pkg.Program.create(st, [g], fusion_kmax=5, tile_qubits=tq, tile_jit=1 if tq > 0 else -1)
                prog.set_timing(True)
                ms = []
                for _ in range(6):
                    prog.run()
                    ms.append(sum(x[0] for x in prog.timings()))
                prog.destroy()
                m = float(np.median(ms[1:]))
                by = 32.0 * frac * (1 << n)
                print(json.dumps({"kind": kind, "k": k, "placement": place, "targets": t, "mode": mode, "n": n,
                                  "ms": round(m, 4), "gbs": round(by / (m * 1e-3) / 1e9, 1),
                                  "frac": round(by / (m * 1e-3) / 1e9 / peak, 3)}), flush=True)
