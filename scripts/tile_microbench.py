"""Tile-pass microbenchmark (developer tool, GPU only): one pass of k Hadamards on high
physical bits with tile T, i.e. W = T - k low contiguous bits per tile; plus a torch copy."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2402_08136_b200 as pkg  # noqa: E402

n = int(os.environ.get("N", "30"))
H = np.array([[1, 1], [1, -1]], complex) / np.sqrt(2)
st = pkg.State(n)
x = torch.empty(2 ** n * 2, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(2):
    y.copy_(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"torch copy 2^{n} c128: {ms:.3f} ms  {2 * 16 * 2**n / ms / 1e6:.0f} GB/s")
del x, y
for T in (10, 11, 12, 13):
    for k in range(0, T - 0, 1):
        gates = [{"kind": "dense", "targets": [n - 1 - i], "data": H} for i in range(k)] or \
                [{"kind": "diagonal", "targets": [0], "data": np.array([1, 1], complex)}]
        prog = pkg.Program.create(st, gates, fusion_kmax=1 if k else 0, tile_qubits=T)
        prog.set_timing(True)
        for _ in range(3):
            prog.run()
        t = prog.timings()
        tt = [x for x in t if x[1] == 5]
        ms = tt[0][0]
        print(f"T={T:2d} k={k:2d} W={T - k:2d}: {ms:8.3f} ms  {32 * 2**n / ms / 1e6:7.0f} GB/s  steps={len(t)}")
        prog.destroy()
for k in (1, 2, 3, 4, 5):
    g = np.random.default_rng(0)
    from workloads import synthetic
    U = synthetic.haar_unitary(k, g)
    for tq in ([0, 1, 2, 3, 4][:k], list(range(n - k, n))):
        for mode in (-1, 12):
            prog = pkg.Program.create(st, [{"kind": "dense", "targets": tq, "data": U}], fusion_kmax=0, tile_qubits=mode)
            prog.set_timing(True)
            for _ in range(3):
                prog.run()
            ms = prog.timings()[0][0]
            print(f"dense k={k} t={tq} tile={mode}: {ms:.3f} ms {32 * 2**n / ms / 1e6:.0f} GB/s")
            prog.destroy()
