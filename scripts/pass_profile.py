"""Per-step CUDA-event timing of one HHL program (developer tool, GPU only).

    python scripts/pass_profile.py [--config S30] [--kmax 4] [--tile 12] [--reps 2]
Prints each scheduled step (kind, ops, ms, GB/s of its HBM bytes) and the total.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="S30")
ap.add_argument("--kmax", type=int, nargs="+", default=[4])
ap.add_argument("--tile", type=int, nargs="+", default=[12])
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--qpe", type=int, nargs="+", default=[0])
ap.add_argument("--jit", type=int, nargs="+", default=[0])
ap.add_argument("--dk", type=int, nargs="+", default=[0])
ap.add_argument("--fold", type=int, nargs="+", default=[0])
ap.add_argument("--verbose", action="store_true")
a = ap.parse_args()
A, b, nc = configs.get(a.config)
st = pkg.State(configs.n_qubits(a.config))
import itertools  # noqa: E402
for q, k, T, J, DK, FO in itertools.product(a.qpe, a.kmax, a.tile, a.jit, a.dk, a.fold):
    if True:
        prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, fusion_kmax=k, tile_qubits=T, qpe_mode=q, tile_jit=J, diag_kmax=DK, init_fold=FO)
        prog.set_timing(True)
        for _ in range(a.reps):
            prog.run()
            t = prog.timings(with_flops=True)
        dump = prog.dump().splitlines()
        heads = [ln for ln in dump if not ln.startswith(("  ", " |"))]
        total = sum(x[0] for x in t)
        import time as _t
        print(f"== {a.config} qpe={q} kmax={k} tile={T} jit={J} dk={DK} fold={FO}: {len(t)} steps, {prog.report['n_fused']} fused ops, "
              f"total {total:.1f} ms")
        if a.verbose:
            for (ms, kind, by, la, fl), h in zip(t, heads):
                roof = max(by / 6533.2e9, fl / (148 * 64 * 2 * 1.965e9)) * 1e3
                print(f"   {ms:9.3f} ms  {by / ms / 1e6 if ms > 0 else 0:8.1f} GB/s  {fl / 1e9:8.1f} GF  "
                      f"roof {roof:6.2f} ms  {h[:80]}")
        prog.destroy()
