"""Host race / bounds / barrier check of the generated tile kernels (compute-sanitizer stand-in; the
tool is closed on the GPU pool). Writes a report (default profiles/r02_jit_racecheck.txt).

    python scripts/jit_racecheck.py [out]
Cases: random circuits (dense / controlled / diagonal / swap mixes, 3-qubit ops) at T = 7..12 and the
C1-C3 / S18 HHL programs (bench, default-JIT and textbook options), each emulated from its initial
state and compared with the oracle; plus every S30 bench pass at full launch size on a prefix of its
tiles (checks only). See tests/jit_emulator.py for what is checked.
"""
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import jit_emulator as emu  # noqa: E402
import paper_2402_08136_b200 as pkg  # noqa: E402
from oracle import hhl as ohhl  # noqa: E402
from oracle import sim  # noqa: E402
from workloads import configs, synthetic  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_jit_racecheck.txt")
lines = []


def log(s):
    print(s, flush=True)
    lines.append(s)


def export(fn):
    d = tempfile.mkdtemp(prefix="emu_")
    os.environ["HHLSV_EMU_DIR"] = d
    try:
        txt = fn()
    finally:
        os.environ.pop("HHLSV_EMU_DIR", None)
    return d, txt


def summ(reps):
    keys = ("races", "oob", "double_writes", "sync_mismatch")
    return {k: sum(r[k] for r in reps) for k in keys}, len(reps)


t0 = time.time()
log("# host race / bounds / barrier check of the NVRTC tile kernels (tests/jit_emulator.py), round 2")
log("# columns: case | passes | races oob double_writes sync_mismatch | max|psi - oracle|")
bad = 0
n = 12
for kinds in [("controlled", "diagonal"), ("dense", "controlled"), ("dense", "diagonal", "swap")]:
    for T in (7, 8, 9, 10, 11, 12):
        gates = synthetic.random_circuit(n, 40, seed=700 + T, kinds=kinds, kmax=3)
        psi0 = synthetic.random_state(n, T)
        d, txt = export(lambda: pkg.schedule_dump(n, gates, fusion_kmax=2, tile_qubits=T, tile_jit=1)[0])
        out, reps = emu.run_program(d, psi0)
        err = float(np.abs(emu.to_logical(out, emu.final_map(txt)) - sim.run(gates, n, psi0)).max())
        c, k = summ(reps)
        bad += sum(c.values()) + (err > 1e-12)
        log(f"random n=12 kinds={'+'.join(kinds)} T={T} | {k} | {c['races']} {c['oob']} {c['double_writes']} "
            f"{c['sync_mismatch']} | {err:.2e}")
for name in ("C1", "C2", "C3p", "C3", "S18"):
    A, b, nc = configs.get(name)
    xo, po, psi_o, p = ohhl.solve(A, b, nc)
    for label, opts in (("bench", configs.BENCH_OPTS), ("bench + fused marginal", dict(configs.BENCH_OPTS, fused_marginal=1)),
                        ("jit T=9", dict(tile_jit=1, tile_qubits=9)),
                        ("textbook k2 T=10", dict(tile_jit=1, tile_qubits=10, fusion_kmax=2)),
                        ("textbook k4 T=12 (wide-run products)", dict(tile_jit=1, tile_qubits=12, fusion_kmax=4, qpe_mode=0))):
        d, txt = export(lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, **opts)[0])
        try:
            out, reps = emu.run_program(d, np.full(1 << p.n, np.nan + 1j * np.nan))
        except RuntimeError as e:
            log(f"{name} {label} | not emulated: {str(e).splitlines()[0]}")
            continue
        err = float(np.abs(emu.to_logical(out, emu.final_map(txt)) - psi_o).max())
        if "red" in reps[-1]:      # fused marginal of the last pass vs the oracle's P(ancilla = 0 / 1)
            h = 1 << (p.n - 1)
            want = (np.sum(np.abs(psi_o[:h]) ** 2), np.sum(np.abs(psi_o[h:]) ** 2))
            err = max(err, float(np.abs(np.array(reps[-1]["red"]) - want).max()))
        c, k = summ(reps)
        bad += sum(c.values()) + (err > 1e-12)
        log(f"HHL {name} ({p.n} q) {label} | {k} | {c['races']} {c['oob']} {c['double_writes']} {c['sync_mismatch']} "
            f"| {err:.2e}")
A, b, nc = configs.get("S30")
d, txt = export(lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, **configs.BENCH_OPTS)[0])
reps = emu.check_full_size(d, 1 << 30, tiles=3)
for r in reps:
    bad += r["races"] + r["oob"] + r["double_writes"] + r["sync_mismatch"]
    log(f"S30 bench pass {r['pass_index']} full launch ({r['launch_tiles']} tiles, {r['nthr']} threads, "
        f"{r['smem']} B smem), first {r['tiles']} tiles | 1 | {r['races']} {r['oob']} {r['double_writes']} "
        f"{r['sync_mismatch']} | n/a (checks only)")
A, b, nc = configs.get("S33")       # sharded over 8 ranks: rank 0's passes (lifted bits, spill fallback)
d, txt = export(lambda: pkg.hhl_schedule_dump(A, b, clock_qubits=nc, world=8, **configs.BENCH_OPTS)[0])
reps = emu.check_full_size(d, 1 << 30, tiles=3)
for r in reps:
    bad += r["races"] + r["oob"] + r["double_writes"] + r["sync_mismatch"]
    log(f"S33/8 rank-0 pass {r['pass_index']} full launch ({r['launch_tiles']} tiles, {r['nthr']} threads, "
        f"{r['smem']} B smem), first {r['tiles']} tiles | 1 | {r['races']} {r['oob']} {r['double_writes']} "
        f"{r['sync_mismatch']} | n/a (checks only)")
log(f"# total findings: {bad} ({time.time() - t0:.0f} s)")
with open(out_path, "w") as f:
    f.write("\n".join(lines) + "\n")
sys.exit(1 if bad else 0)
