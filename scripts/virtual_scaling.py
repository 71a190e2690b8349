"""Weak-scaling projection from ONE B200 (the pool has one GPU per call): the S31/S32/S33 programs run as
2/4/8 in-process virtual shards (the same per-rank schedule, rank-resolved kernels, lifted / slot-range
passes and exchange packing as the NCCL path; exchanges are device copies), timed per step with CUDA
events. Per-rank compute = the shards' pass time / world (they run one after another here). The exchange
is modelled at the guide's measured 770 GB/s peer bandwidth per direction, pipelined with the pass before
it (the engine sends each slot while computing the next): exposed = max(that pass, transfer).

    python scripts/virtual_scaling.py > profiles/r02_virtual_scaling.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402

NVLINK = 770e9


def run(cfg, world):
    A, b, nc = configs.get(cfg)
    st = pkg.State(configs.n_qubits(cfg), world=world) if world > 1 else pkg.State(configs.n_qubits(cfg))
    prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, **configs.BENCH_OPTS)
    for _ in range(2):
        prog.run()
    prog.set_timing(True)
    best = None
    for _ in range(3):
        prog.run()
        t = prog.timings(with_flops=True)
        tot = sum(x[0] for x in t)
        if best is None or tot < best[0]:
            best = (tot, t)
    prog.destroy()
    st.destroy()
    pkg.trim_memory()
    return best[1]


t30 = run("S30", 1)
T30 = sum(x[0] for x in t30)
print(json.dumps({"workload": "S30", "world": 1, "ms": T30, "steps": [round(x[0], 3) for x in t30]}), flush=True)
for cfg, world in (("S31", 2), ("S32", 4), ("S33", 8)):
    # the same circuit on ONE GPU (S33 = 128 GiB fits in 180 GB): separates the sharding overhead from the
    # circuit's growth with the clock register (per-amplitude work rises with n_clock)
    t1 = run(cfg, 1)
    T1 = sum(x[0] for x in t1)
    t = run(cfg, world)
    passes = [(ms / world, kind, by) for ms, kind, by, la, fl in t if kind != 6]
    ex = [(ms, by) for ms, kind, by, la, fl in t if kind == 6]
    per_rank = [round(p[0], 3) for p in passes]
    proj = sum(p[0] for p in passes)
    xfer = 0.0
    if ex:
        # bytes each rank sends = half of the exchange's (send + receive) bytes per shard
        xfer = (ex[0][1] / world) / 2 / NVLINK * 1e3
        kinds = [k for _, k, _, _, _ in t]
        i = kinds.index(6)
        before = t[i - 1][0] / world if i > 0 else 0.0
        proj += max(before, xfer) - before
    print(json.dumps({"workload": cfg, "world": world, "per_rank_pass_ms": per_rank,
                      "virtual_exchange_ms": [round(e[0], 3) for e in ex], "modelled_nvlink_ms": round(xfer, 3),
                      "projected_ms_per_rank": round(proj, 3), "projected_weak_scaling_E": round(T30 / proj, 3),
                      "one_gpu_ms": round(T1, 3), "projected_speedup_vs_one_gpu": round(T1 / proj, 3),
                      # SURVEY §8(d) "pass-normalized E": the same circuit on 1 GPU vs world GPUs
                      "projected_same_circuit_efficiency": round(T1 / proj / world, 3),
                      "how": "per-rank passes measured (virtual shards, one GPU), exchange modelled at 770 GB/s "
                             "and overlapped with the pass before it"}), flush=True)
