"""Time hhl_solve end to end with stage markers (developer tool, GPU): HHLSV_PROFILE=1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402
A, b, nc = configs.get("S30")
for i in range(3):
    t = time.perf_counter()
    x, rep = pkg.hhl_solve(A, b, clock_qubits=nc, qpe_mode=1, fusion_kmax=1, tile_qubits=12)
    print(f"solve {i}: {time.perf_counter() - t:.3f} s  frontend {rep['t_frontend_s']*1e3:.1f} ms  sim {rep['t_sim_s']*1e3:.1f} ms", flush=True)
