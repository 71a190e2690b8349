import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2402_08136_b200 as pkg
from workloads import configs
A, b, nc = configs.get("B30")
flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device="cuda")
for dev in (None, 0):
    for fl in (False, True):
        ts = []
        for i in range(6):
            if fl: flush.fill_(float(i))
            torch.cuda.synchronize()
            t = time.perf_counter()
            kw = dict(device=0) if dev is not None else {}
            x, rep = pkg.hhl_solve(A, b, clock_qubits=nc, **configs.BENCH_OPTS, **kw)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        print("device", dev, "flush", fl, [round(v, 2) for v in ts])
