"""Padded stress circuit P_n timing on one GPU: one JSON line.

    python scripts/stress_bench.py [--n 30] [--kmax 2] [--steps 5]
C3's 15-qubit textbook HHL gate list on a seeded random injective qubit map + 8 brickwork layers on the
pad qubits, through the generic gate-list API (sv_program_create: fusion, tile scheduling, NVRTC passes).
Timed with CUDA events after 3 warm-up runs; the state (16 GiB at n = 30) is far larger than L2.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs, synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--kmax", type=int, default=2)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--profile", action="store_true", help="also print per-step times and the schedule to stderr")
a = ap.parse_args()
from oracle import hhl as ohhl  # noqa: E402  (input generation: the 15-qubit logical list)
A, b, nc = configs.get("C3")
p = ohhl.plan(A, b, nc)
gates, qmap, pad = synthetic.padded_circuit(ohhl.build(p), p.n, a.n)
st = pkg.State(a.n)
prog = pkg.Program.create(st, gates, fusion_kmax=a.kmax, tile_qubits=12, tile_jit=1)
for _ in range(3):
    st.reset()
    prog.run()
torch.cuda.synchronize()
ms = []
for _ in range(a.steps):
    st.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    prog.run()
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
t = sorted(ms)[len(ms) // 2]
if a.profile:
    prog.set_timing(True)
    st.reset()
    prog.run()
    for i, (m, kind, by, la, fl) in enumerate(prog.timings(with_flops=True)):
        print(f"step {i}: kind {kind} {m:8.3f} ms {by / 1e9:6.2f} GB {fl / 1e9:8.1f} GF", file=sys.stderr)
    print(prog.dump(), file=sys.stderr)
rep = prog.report
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({"workload": f"P{a.n}", "n_logical_gates": len(gates), "n_fused": rep["n_fused"],
                  "n_passes": rep["n_passes"], "fusion_kmax": a.kmax, "ms_per_run": t,
                  "hbm_bytes": rep["pass_bytes"], "hbm_gbs": rep["pass_bytes"] / (t * 1e-3) / 1e9,
                  "frac_of_peak": rep["pass_bytes"] / (t * 1e-3) / 1e9 / peak, "stats": prog.stats()}))
