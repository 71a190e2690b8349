"""Time hhl_solve end to end with stage markers (developer tool, GPU): HHLSV_PROFILE=1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402
A, b, nc = configs.get(sys.argv[1] if len(sys.argv) > 1 else "S30")
for i in range(5):
    t = time.perf_counter()
    x, rep = pkg.hhl_solve(A, b, clock_qubits=nc, **configs.BENCH_OPTS)
    print(f"solve {i}: {(time.perf_counter() - t) * 1e3:.1f} ms  frontend {rep['t_frontend_s']*1e3:.1f} ms  "
          f"sim {rep['t_sim_s']*1e3:.1f} ms", file=sys.stderr, flush=True)
