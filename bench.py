#!/usr/bin/env python
"""HHL state-vector hot-path benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
    python bench.py --table1        # Table 1 / configs[0..2] regime: one line per small config

Workload (default): the synthetic HHL-shaped circuit of BASELINE.json configs[3] (S30: the IEEE
14-bus DC system padded to 16x16, n_c = 25 clock qubits, 30 qubits = 16 GiB of complex128) at
N = 1; at N GPUs the weak-scaled S(30 + log2 N) circuit sharded by global qubits (configs[4]:
31/32/33 qubits on 2/4/8 GPUs, 2^30 amplitudes per GPU).

A step = one pass of the whole hot path over the resident state: product-state init (a3), every
fused op of the circuit (a4-a7, tile passes), the post-selection readout and recovery (a8, a9).

value      = fused-gate GB/s: the HBM bytes the step's passes move (read + write, 16 B per
             amplitude, summed over ranks) / step time. A real bandwidth: its fraction of the
             measured HBM copy peak is the metric's "fraction of HBM peak".
ms_per_step = the HHL circuit simulation time (the metric's "circuit sim time").
e2e        = the same bytes / the time of hhl_solve() with HOST A, b -> HOST x (front end, uploads,
             state allocation, simulation, readout, D2H inside the timed region).
The CPU oracle (oracle/, test infrastructure) runs ONLY in the cpu_baseline leg (rank 0, N = 1)
and in --impl reference; it also yields config.parity_max_abs (the bench program vs eq. CF).
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
# FP64 vector peak of the B200, DERIVED: 148 SMs x 64 FP64 FMA lanes x 2 flop x 1.965 GHz.
# profiles/r02_fp64_peak.json holds the DFMA microbenchmark measured on the box (used when present).
FP64_PEAK_DERIVED = 148 * 64 * 2 * 1.965e9
L2_FLUSH_BYTES = 512 << 20              # > 126 MB L2


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["dfma_tflops"]) * 1e12, f"measured DFMA microbenchmark ({d.get('when', 'r02')})"
    except Exception:
        return FP64_PEAK_DERIVED, "derived: 148 SMs x 64 FP64 FMA lanes x 2 flop x 1.965 GHz"


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


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model, os.cpu_count()


# ------------------------------------------------------------------ oracle legs
def gate_bytes(g: dict, n: int) -> float:
    """SURVEY §8(d) bytes one unfused logical gate moves when applied as its own pass."""
    if g["kind"] == "swap":
        return 32.0 * 2 ** n
    if g["kind"] == "controlled":
        return 32.0 * 2 ** n / 2 ** len(g["controls"])
    return 32.0 * 2 ** n


def textbook_bytes(cfg: str) -> tuple[float, int]:
    """Bytes of the config's textbook HHL circuit (Fig. 5) as unfused logical gates, each its own
    pass (oracle builder only): the 'gate-equivalent' numerator of config.textbook_equiv_gbs."""
    from oracle import hhl as ohhl
    from workloads import configs
    A, b, nc = configs.get(cfg)
    p = ohhl.plan(A, b, nc)
    gates = ohhl.build(p)
    return float(sum(gate_bytes(g, p.n) for g in gates)), len(gates)


def oracle_sample(cfg: str, budget_s: float):
    """Time the CPU oracle (as it stands, all host threads) on a bounded sample of the workload:
    the first logical gates of the config's unfused HHL list applied to a 2^n host state until
    ~budget_s. value = the bytes those gate loops move (16 B read + 16 B written per visited
    amplitude) / time; extrapolated_full_s = the whole circuit at the sample's rate."""
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
    total = sum(gate_bytes(g, n) for g in gates)
    psi = sim.zero_state(n)
    t0 = time.perf_counter()
    done, nbytes = 0, 0.0
    for g in gates:
        sim.apply_gate(psi, n, g)
        done += 1
        nbytes += gate_bytes(g, n)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    model, ncpu = host_cpu()
    return {"value": nbytes / dt / 1e9, "unit": "GB/s", "cores": sim.n_threads(), "kind": "oracle",
            "sample": f"first {done} of {len(gates)} logical gates of the {cfg}-shaped HHL circuit, unfused, "
                      f"on a 2^{n} complex128 host state ({dt:.1f} s)",
            "seconds": dt, "gates": done, "n": n,
            "extrapolated_full_s": dt * total / nbytes, "host_cpu": model, "host_threads": ncpu}


def parity_s30(pkg, st, A, b, nc, cfg, opts):
    """config.parity_max_abs: the bench program (same options, same kernels) vs eq. CF on one whole
    clock block of 2^8 clock values x 16 system x 2 ancilla (k_high 0: holds the post-selected slice).
    'oracle_eig' builds it with the oracle's eigendecomposition (bit-identical phases: the engine's
    1e-10 bar); 'product_eig' is the program bench.py timed (own Jacobi eigensolver; bounded by the
    front-end tolerance of DESIGN.md §5)."""
    from oracle import closed_form as cf
    from oracle import hhl as ohhl
    p = ohhl.plan(A, b, nc)
    B = 8
    ref = cf.block_amplitudes(p, [0], B)[:, 0]
    out = {}
    for eig in ("oracle", "product"):
        kw = dict(opts)
        if eig == "oracle":
            kw["eig"] = (p.lam, p.V)
        prog = pkg.HHLProgram.build(st, A, b, **kw)
        prog.run()
        got = np.stack([st.read(a << (p.n - 1), (1 << B) << p.n_b).reshape(1 << B, 1 << p.n_b) for a in (0, 1)])
        out[f"{eig}_eig"] = float(np.abs(got - ref).max())
        prog.destroy()
    out["amplitudes"] = int(ref.size)
    out["tol_product_eig"] = max(1e-10, 2 * np.pi * (1 << p.n_c) * 8 * np.finfo(float).eps * float(np.max(np.abs(p.phi))))
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config or ("S30" if args.gpus == 1 else f"S{30 + int(math.log2(args.gpus))}")
    vals = []
    per_step = max(3.0, 60.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        r = oracle_sample(cfg, per_step)
        if i >= args.warmup:
            vals.append(r)
    v = float(np.mean([r["value"] for r in vals]))
    ms = float(np.mean([r["seconds"] for r in vals])) * 1e3
    last = vals[-1]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg, "sample": last["sample"],
                       "extrapolated_full_circuit_s": last["extrapolated_full_s"]},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"], "host_cpu": last["host_cpu"]},
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
    n = configs.n_qubits(cfg)
    small = (16 << (n - int(math.log2(world)))) < (256 << 20)     # state fits in L2: flush between steps
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda") if small else None

    st = pkg.State(n, world=world, rank=rank, device=local, nccl_id=nccl_id)
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
    per_pass = {}
    peak_gbs, peak_src = measured_peaks()
    fp64_pk, fp64_src = fp64_peak()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with clocks:
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))                # L2 flush outside the timed span of the step
            evs[i][0].record(stream)
            x, ps = step()                          # readout synchronises the stream
            evs[i][1].record(stream)
            for si, (ms, kind, by, la, fl) in enumerate(prog.timings(with_flops=True)):
                if kind == 5:        # per tile pass (step index): time, bytes, flops over the timed steps
                    q = per_pass.setdefault(si, [0.0, 0, by, fl])
                    q[0] += ms
                    q[1] += 1
                d = per_kind.setdefault(kind, [0.0, 0, 0.0, 0.0, 0.0])
                d[0] += ms
                d[1] += 1
                d[2] += by
                d[3] += fl
                d[4] += max(by / (peak_gbs * 1e9), fl / fp64_pk) * 1e3
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_step = float(sum(e0.elapsed_time(e1) for e0, e1 in evs)) / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    prog.set_timing(False)
    step_bytes = float(rep["pass_bytes"]) * world          # HBM bytes of all ranks' passes
    value = step_bytes / (ms_step * 1e-3) / 1e9

    # dominant kernel (largest total time) and its roofline
    kind_exchange = 6
    kind_names = pkg.sv.STEP_KINDS
    dom = max(((k, v) for k, v in per_kind.items() if k != kind_exchange), key=lambda kv: kv[1][0])
    dom_kind, (dom_ms, dom_n, dom_bytes, dom_flops, dom_roof_ms) = dom
    dom_avg = dom_ms / max(1, dom_n)
    bytes_per_launch = dom_bytes / max(1, dom_n)
    achieved = bytes_per_launch / (dom_avg * 1e-3) / 1e9
    traffic = None
    try:   # DRAM bytes per launch of the dominant kernel from this round's committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("kernel") == "hhlsv_tile" and kind_names[dom_kind] == "tile" and tr.get("workload") == cfg:
            traffic = float(tr["dram_bytes_per_launch"])
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s", "frac": achieved / peak_gbs,
                "traffic": traffic, "kernel": "hhlsv_tile" if kind_names[dom_kind] == "tile" else kind_names[dom_kind],
                "avg_launch_ms": dom_avg, "launches_per_step": dom_n / args.steps,
                "bytes_per_launch": bytes_per_launch, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                "share_of_step": dom_ms / args.steps / ms_step,
                # the tile passes also carry FP64 work: per launch the roofline time is
                # max(bytes / HBM peak, flops / FP64 peak); combined_frac = that / measured time
                "fp64_tflops_achieved": dom_flops / (dom_ms * 1e-3) / 1e12,
                "fp64_peak_tflops": fp64_pk / 1e12, "fp64_peak_source": fp64_src,
                "combined_frac": dom_roof_ms / dom_ms,
                # each tile pass of the step (north_star: "a 30-qubit fused pass at >= 70 % of HBM")
                "passes": [{"step": si, "ms": q[0] / q[1], "bytes": q[2],
                            "gbs": q[2] / (q[0] / q[1] * 1e-3) / 1e9,
                            "frac": q[2] / (q[0] / q[1] * 1e-3) / 1e9 / peak_gbs,
                            "fp64_tflops": q[3] / (q[0] / q[1] * 1e-3) / 1e12} for si, q in sorted(per_pass.items())]}

    nvlink = None
    if kind_exchange in per_kind:      # global-qubit swaps: bytes each rank sends + receives per exchange
        xms, xn, xby = per_kind[kind_exchange][:3]
        xby = xby / max(1, xn)
        nvlink = {"exchanges_per_step": xn // max(1, args.steps), "ms_per_exchange": xms / max(1, xn),
                  "bytes_per_exchange": xby, "gbs": xby / (xms / max(1, xn) * 1e-3) / 1e9 if xms > 0 else None,
                  "share_of_step": xms / args.steps / ms_step}

    # shot-sampling readout on the final state: 10^5 shots (N=1; sv_sample is single-rank)
    sample = None
    if world == 1 and not small:
        try:
            st.sample(1000, seed=1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st.sample(100000, seed=2402)
            ts = time.perf_counter() - t0
            nb = 16.0 * (1 << n)
            sample = {"shots": 100000, "ms": ts * 1e3, "state_read_gbs": nb / ts / 1e9}
        except Exception as exc:
            sample = {"error": str(exc)[:200]}

    # e2e through the public API with host buffers, right after the timed region (the GPU still at
    # speed; the bench state stays allocated: 2 x 16 GiB fit in HBM)
    e2e = None
    if not args.no_e2e:
        # N = 1: hhl_solve (host A, b -> host x; creates and frees its own state). N > 1: a sharded state
        # is a session object (its NCCL communicator is created once, like the process group): each solve
        # builds the program from host A, b on it (front end + uploads), runs it and reads x back.
        est = None
        if world > 1:
            prog.destroy()
            st.destroy()
            prog = st = None
            idt2 = torch.zeros(128, dtype=torch.uint8, device="cuda")      # a fresh communicator id
            if rank == 0:
                idt2.copy_(torch.frombuffer(bytearray(pkg.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt2, 0)
            est = pkg.State(n, world=world, rank=rank, device=local, nccl_id=bytes(idt2.cpu().numpy().tobytes()))
        times = []
        for i in range(max(1, args.e2e_steps) + 2):         # 2 untimed warm-up solves
            if world > 1:
                dist.barrier()
            if flush is not None:
                flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if est is None:
                xe, r2 = pkg.hhl_solve(A, b, world=world, rank=rank, device=local, **opts)
            else:
                ep = pkg.HHLProgram.build(est, A, b, **opts)
                ep.run()
                xe, _ = ep.readout()
                r2 = dict(ep.report)
                ep.destroy()
            torch.cuda.synchronize()
            if i > 1:
                times.append(time.perf_counter() - t0)
        if est is not None:
            est.destroy()
        te = float(np.median(times))               # median: robust to one-off driver stalls
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": step_bytes / te / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(r2["h2d_bytes"] + A.nbytes + b.nbytes),
               "d2h_bytes_per_step": int(r2["d2h_bytes"]), "seconds": te,
               "t_frontend_s": r2["t_frontend_s"], "t_sim_s": r2["t_sim_s"],
               "p_anc1": r2["p_anc1"]}

    # ---- cpu_baseline leg (rank 0, N = 1): the oracle timed on this host, and the parity check
    cpu = None
    parity = None
    textbook = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(cfg, args.cpu_budget)
        tb, tn = textbook_bytes(cfg)
        textbook = {"logical_gates": tn, "bytes": tb, "equiv_gbs": tb / (ms_step * 1e-3) / 1e9}
        if cfg == "S30" and not args.no_parity:
            parity = parity_s30(pkg, st, A, b, nc, cfg, opts)

    if prog is not None:
        prog.destroy()
        st.destroy()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg, "n_qubits": rep["n_total"], "n_data": rep["n_data"],
                           "n_clock": rep["n_clock"], "system": configs.describe(cfg),
                           "n_logical_gates": rep["n_logical"], "n_ops_executed": rep["n_fused"],
                           "n_passes": rep["n_passes"], "fusion_kmax": args.kmax, "tile_qubits": args.tile,
                           "qpe_mode": ["textbook", "eigenbasis"][args.qpe], "tile_jit": args.jit,
                           "l2": ("L2 flushed (512 MiB write) before every step" if small
                                  else f"state ({16 << (n - int(math.log2(world))) >> 20} MiB/GPU) >> 126 MB L2; no flush"),
                           "hhl_circuit_time_ms": ms_step, "p_success": ps,
                           "hbm_bytes_per_step": step_bytes, "hbm_frac_of_peak": value / peak_gbs,
                           "textbook_unfused": textbook, "parity_max_abs": parity,
                           # context only (another machine, end to end incl. Python): Table 1
                           "paper_sv_sim_a100_s": {"C3p": 13.0, "B30": 234.0}.get(cfg)},
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--table1", action="store_true", help="one line per small config (C1 C2 C3p C3 B30)")
    from workloads.configs import BENCH_OPTS
    ap.add_argument("--kmax", type=int, default=BENCH_OPTS["fusion_kmax"])
    ap.add_argument("--tile", type=int, default=BENCH_OPTS["tile_qubits"])
    ap.add_argument("--qpe", type=int, default=BENCH_OPTS["qpe_mode"],
                    help="0 textbook c-U chain, 1 eigenbasis rewrite (SURVEY f2)")
    ap.add_argument("--jit", type=int, default=BENCH_OPTS["tile_jit"],
                    help="tile pass specialisation: 0 auto, 1 on, -1 off")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.table1:
        rc = 0
        for c in ("C1", "C2", "C3p", "C3", "B30"):
            a2 = argparse.Namespace(**vars(args))
            a2.config = c
            a2.cpu_budget = min(args.cpu_budget, 5.0)
            rc |= run_reference(a2) if args.impl == "reference" else run_ours(a2)
        sys.exit(rc)
    sys.exit(run_reference(args) if args.impl == "reference" else run_ours(args))


if __name__ == "__main__":
    main()
