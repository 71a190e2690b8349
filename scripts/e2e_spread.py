"""hhl_solve wall times, one per line, after the bench program of the same config is resident (the
bench's e2e situation): shows the spread of the e2e number (developer tool, GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "S30"
A, b, nc = configs.get(cfg)
opts = dict(configs.BENCH_OPTS, clock_qubits=nc)
st = pkg.State(configs.n_qubits(cfg))
prog = pkg.HHLProgram.build(st, A, b, **opts)
for _ in range(5):
    prog.run()
    prog.readout()
ts = []
for i in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, r = pkg.hhl_solve(A, b, **opts)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{cfg} solve {i}: {ts[-1]:.2f} ms (front end {r['t_frontend_s'] * 1e3:.2f}, sim {r['t_sim_s'] * 1e3:.2f})",
          flush=True)
