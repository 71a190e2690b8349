"""Measured vs predicted (a2 cost model) time per fusion width (GPU, developer tool): one line per case.

    python scripts/cost_model_check.py [--config S26]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="S26")
a = ap.parse_args()
A, b, nc = configs.get(a.config)
st = pkg.State(configs.n_qubits(a.config))
for tiles, ks in ((12, (1, 2, 3, 4)), (-1, (1, 2, 3, 4, 5))):
    auto = pkg.hhl_schedule_dump(A, b, clock_qubits=nc, qpe_mode=1, tile_qubits=tiles, tile_jit=1 if tiles > 0 else 0)[1]
    for k in ks:
        prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, qpe_mode=1, tile_qubits=tiles, fusion_kmax=k,
                                    tile_jit=1 if tiles > 0 else 0)
        for _ in range(2):
            prog.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            prog.run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(json.dumps({"config": a.config, "tile_qubits": tiles, "fusion_kmax": k, "measured_ms": sorted(ts)[2],
                          "model_ms": prog.report["model_ms"], "passes": prog.report["n_passes"],
                          "auto_choice": auto["fusion_kmax_used"]}), flush=True)
        prog.destroy()
