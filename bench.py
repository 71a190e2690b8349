#!/usr/bin/env python
"""HHL state-vector hot-path benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload: the synthetic HHL-shaped circuit of BASELINE.json configs[3] (S30: the IEEE
14-bus DC system padded to 16x16, n_c = 25 clock qubits, 30 qubits = 16 GiB of complex128)
at N = 1; at N GPUs the weak-scaled S(30 + log2 N) circuit sharded by global qubits
(configs[4]: 31/32/33 qubits on 2/4/8 GPUs, 2^30 amplitudes per GPU).

A step = one pass of the whole hot path over the resident state: product-state init (a3),
every fused op of the circuit (a4-a7, tile passes), and the post-selection readout (a8).
value  = fused-gate GB/s = CANONICAL algorithmic bytes / step time. Canonical bytes: the paper's
         textbook HHL circuit for the config (Fig. 5), fused with the default structure-preserving
         fusion (k_max 4, diagonals <= 12 qubits; S30 -> 168 fused ops), each op
         counted at its SURVEY §8(d) bytes (32·2^n per dense/diagonal/recip op, 32·2^(n-c) per
         controlled op). Fixed per workload: independent of how this engine fuses or schedules.
e2e    = the same metric through hhl_solve() with HOST A, b -> HOST x (front end, uploads,
         state allocation, simulation, readout, D2H all inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HHL circuit sim time & fused-gate GB/s (fraction of HBM peak) at 1/2/4/8 B200"
FP64_PEAK = 148 * 64 * 2 * 1.965e9          # flop/s, derived from unit counts and the max SM clock


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------ oracle arm
def canonical_bytes(cfg: str) -> tuple[float, int]:
    """Canonical algorithmic bytes of the config's HHL circuit (module docstring) and its fused-op
    count: host-only planning through the C ABI (hhl_schedule_dump), no GPU."""
    import paper_2402_08136_b200 as pkg
    from workloads import configs
    A, b, nc = configs.get(cfg)
    _, r = pkg.hhl_schedule_dump(A, b, clock_qubits=nc, qpe_mode=0, fusion_kmax=4, diag_kmax=12, tile_qubits=-1)
    return float(r["alg_bytes"]), int(r["n_fused"])


def oracle_sample(cfg: str, budget_s: float, max_n: int = 30):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: the first
    gates of the config's logical HHL list applied to a 2^n host state, until ~budget_s."""
    from oracle import hhl as ohhl
    from oracle import sim
    from workloads import configs
    A, b, nc = configs.get(cfg)
    p = ohhl.plan(A, b, nc)
    gates = ohhl.build(p)
    n = p.n
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    while n > 20 and (16 << n) * 1.5 > avail:
        n -= 1
    if n != p.n:   # host cannot hold the state: same gate list shape on fewer clock qubits
        p = ohhl.plan(A, b, n - p.n_b - 1)
        gates = ohhl.build(p)
    def gbytes(g):
        return 32.0 * 2 ** n / (2 ** len(g.get("controls", [])) if g["kind"] == "controlled" else 1)
    total = sum(gbytes(g) for g in gates)
    psi = sim.zero_state(n)
    t0 = time.perf_counter()
    done, nbytes = 0, 0.0
    for g in gates:
        sim.apply_gate(psi, n, g)
        done += 1
        nbytes += gbytes(g)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    # the sampled fraction of the logical circuit, scaled to the canonical bytes of the full-size
    # workload (the same numerator as our arm's value)
    canon, _ = canonical_bytes(cfg)
    return {"value": canon * (nbytes / total) / dt / 1e9, "unit": "GB/s", "cores": sim.n_threads(), "kind": "oracle",
            "sample": f"first {done} of {len(gates)} logical gates of the {cfg}-shaped HHL circuit, unfused, "
                      f"on a 2^{n} complex128 host state ({dt:.1f} s)",
            "seconds": dt, "gates": done, "n": n}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config or ("S30" if args.gpus == 1 else f"S{30 + int(math.log2(args.gpus))}")
    vals = []
    per_step = max(5.0, 60.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        r = oracle_sample(cfg, per_step)
        if i >= args.warmup:
            vals.append(r)
    v = float(np.mean([r["value"] for r in vals]))
    ms = float(np.mean([r["seconds"] for r in vals])) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg, "sample": vals[-1]["sample"]},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": vals[-1]["cores"], "kind": "oracle",
                             "sample": vals[-1]["sample"]},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2402_08136_b200 as pkg
    from workloads import configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(pkg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    cfg = args.config or ("S30" if world == 1 else f"S{30 + int(math.log2(world))}")
    A, b, nc = configs.get(cfg)
    opts = dict(clock_qubits=nc, fusion_kmax=args.kmax, tile_qubits=args.tile, qpe_mode=args.qpe,
                tile_jit=args.jit)
    stream = torch.cuda.current_stream()

    st = pkg.State(configs.n_qubits(cfg), world=world, rank=rank, device=local, nccl_id=nccl_id)
    prog = pkg.HHLProgram.build(st, A, b, **opts)
    rep = prog.report
    stats = prog.stats()

    def step():
        prog.run()
        return prog.readout()

    for _ in range(args.warmup):
        x, ps = step()
    prog.set_timing(True)
    per_kind = {}
    peak_gbs, _ = measured_peaks()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        e0.record(stream)
        for _ in range(args.steps):
            x, ps = step()                      # readout synchronises the stream
            for ms, kind, by, la, fl in prog.timings(with_flops=True):
                d = per_kind.setdefault(kind, [0.0, 0, 0.0, 0.0, 0.0])
                d[0] += ms
                d[1] += 1
                d[2] += by
                d[3] += fl
                # per-launch roofline time: the slower of the HBM and the FP64 bound
                d[4] += max(by / (peak_gbs * 1e9), fl / FP64_PEAK) * 1e3
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_step = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    prog.set_timing(False)
    alg_bytes, canon_ops = canonical_bytes(cfg)   # whole circuit (all ranks' shards), canonical
    value = alg_bytes / (ms_step * 1e-3) / 1e9

    # dominant kernel (largest total time) and its roofline
    peak, peak_src = measured_peaks()
    kind_exchange = 6
    dom = max(((k, v) for k, v in per_kind.items() if k != kind_exchange), key=lambda kv: kv[1][0])
    dom_kind, (dom_ms, dom_n, dom_bytes, dom_flops, dom_roof_ms) = dom
    dom_avg = dom_ms / max(1, dom_n)
    dom_bytes = dom_bytes / max(1, dom_n)          # mean algorithmic bytes per launch (pass 1 writes only)
    achieved = dom_bytes / (dom_avg * 1e-3) / 1e9
    kind_names = pkg.sv.STEP_KINDS
    traffic = None
    try:   # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("kernel") == "hhlsv_tile" and kind_names[dom_kind] == "tile":
            traffic = float(tr["dram_bytes_per_launch"])
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kind_names[dom_kind], "avg_launch_ms": dom_avg,
                "bytes_per_launch": dom_bytes, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                "share_of_step": dom_ms / args.steps / ms_step,
                # the tile passes also carry FP64 work: per launch the roofline time is
                # max(bytes / HBM peak, flops / FP64 peak); combined_frac = roofline time / measured time
                "fp64_tflops_achieved": dom_flops / (dom_ms * 1e-3) / 1e12,
                "fp64_peak_tflops": FP64_PEAK / 1e12,
                "fp64_peak_source": "derived: 148 SMs x 64 FP64 FMA lanes x 2 flop x 1.965 GHz (DESIGN.md §6)",
                "combined_frac": dom_roof_ms / dom_ms}

    nvlink = None
    if kind_exchange in per_kind:      # global-qubit swaps: bytes each rank sends + receives per exchange
        xms, xn, xby = per_kind[kind_exchange][:3]
        xby = xby / max(1, xn)                      # mean bytes per exchange
        nvlink = {"exchanges_per_step": xn // max(1, args.steps), "ms_per_exchange": xms / max(1, xn),
                  "bytes_per_exchange": xby, "gbs": xby / (xms / max(1, xn) * 1e-3) / 1e9 if xms > 0 else None,
                  "share_of_step": xms / args.steps / ms_step}

    # shot-sampling readout on the final S30 state: 10^5 shots (N=1; sv_sample is single-rank)
    sample = None
    if world == 1:
        try:
            st.sample(1000, seed=1)                       # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st.sample(100000, seed=2402)
            ts = time.perf_counter() - t0
            nb = 16.0 * (1 << configs.n_qubits(cfg))      # one read of the state for the block sums
            sample = {"shots": 100000, "ms": ts * 1e3, "state_read_gbs": nb / ts / 1e9}
        except Exception as exc:                          # reported, never fatal for the bench line
            sample = {"error": str(exc)[:200]}

    # e2e through the public API with host buffers (N=1 only: hhl_solve owns its state)
    e2e = None
    if not args.no_e2e:
        if world > 1:
            idt2 = torch.zeros(128, dtype=torch.uint8, device="cuda")
        times = []
        prog.destroy()
        st.destroy()
        for i in range(max(1, args.e2e_steps) + 1):
            nid = None
            if world > 1:
                if rank == 0:
                    idt2.copy_(torch.frombuffer(bytearray(pkg.nccl_unique_id()), dtype=torch.uint8))
                dist.broadcast(idt2, 0)
                nid = bytes(idt2.cpu().numpy().tobytes())
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            xe, r2 = pkg.hhl_solve(A, b, world=world, rank=rank, device=local, nccl_id=nid, **opts)
            torch.cuda.synchronize()
            if i > 0:
                times.append(time.perf_counter() - t0)
        te = float(np.median(times))               # median: robust to one-off driver stalls
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": alg_bytes / te / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(r2["h2d_bytes"] + A.nbytes + b.nbytes),
               "d2h_bytes_per_step": int(r2["d2h_bytes"]), "seconds": te,
               "t_frontend_s": r2["t_frontend_s"], "t_sim_s": r2["t_sim_s"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(cfg, args.cpu_budget)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg, "n_qubits": rep["n_total"], "n_data": rep["n_data"],
                           "n_clock": rep["n_clock"], "system": "IEEE 14-bus DC B (MATPOWER case14), 16x16",
                           "n_logical_gates": rep["n_logical"], "n_fused_ops_canonical": canon_ops,
                           "n_ops_executed": rep["n_fused"],
                           "n_passes": rep["n_passes"], "fusion_kmax": args.kmax, "tile_qubits": args.tile,
                           "qpe_mode": ["textbook", "eigenbasis"][args.qpe], "tile_jit": args.jit,
                           "l2": "state (16 GiB/GPU) >> 126 MB L2; no flush needed",
                           "hhl_circuit_time_ms": ms_step, "p_success": ps,
                           "hbm_pass_gbs": rep["pass_bytes"] / world / (ms_step * 1e-3) / 1e9},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(stats["launches"] + 1), "clocks": clocks.summary()}
        if nvlink:
            line["nvlink"] = nvlink
        if sample:
            line["sample"] = sample
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--kmax", type=int, default=1)
    ap.add_argument("--tile", type=int, default=12)
    ap.add_argument("--qpe", type=int, default=1, help="0 textbook c-U chain, 1 eigenbasis rewrite (SURVEY f2)")
    ap.add_argument("--jit", type=int, default=0, help="tile pass specialisation: 0 auto, 1 on, -1 off")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    sys.exit(run_reference(args) if args.impl == "reference" else run_ours(args))


if __name__ == "__main__":
    main()
