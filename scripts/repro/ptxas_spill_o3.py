"""Standalone reproduction: a generated tile kernel whose registers are capped at 64 (a sub-warp CTA with
the round-1 __launch_bounds__ rule, reproduced with HHLSV_JIT=minb=32; matrices preloaded into registers
with cw=0) spills and computes wrong amplitudes when ptxas optimises at -O3, right ones at -O1 -- while the
host emulation of the SAME source (tests/jit_emulator.py: ASan + UBSan, shared-memory race / bounds /
barrier checks) is clean and matches the oracle.

    python scripts/repro/ptxas_spill_o3.py cpu     # emulate the generated source (no GPU)
    python scripts/repro/ptxas_spill_o3.py gpu     # run it on the B200 at ptxas -O3 and -O1
The product avoids the trigger: __launch_bounds__ counts warps (128 registers for 16-thread CTAs) and small
matrices are constant-bank operands, so the generated kernels do not spill (cuobjdump -res-usage).
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASE = r'''
import os, sys, json
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
import paper_2402_08136_b200 as pkg
from oracle import hhl as ohhl, sim, transpile as tr
from workloads import configs
A, b, nc = configs.get("C1")
t = tr.transpile(ohhl.build(ohhl.plan(A, b, nc)))      # the 2x2 HHL as 1q + CNOT gates
n, T = 10, 8
mode = sys.argv[2]
ref = sim.run(t, n)
if mode == "cpu":
    import jit_emulator as emu
    d = os.environ["HHLSV_EMU_DIR"]
    txt = pkg.schedule_dump(n, t, fusion_mode=1, tile_qubits=T, tile_jit=1)[0]
    out, reps = emu.run_program(d, np.eye(1, 1 << n, dtype=complex)[0])
    err = float(np.abs(emu.to_logical(out, emu.final_map(txt)) - ref).max())
    print(json.dumps({"where": "host emulation", "max_err": err,
                      "checks": [{k: r[k] for k in ("races", "oob", "double_writes", "sync_mismatch")} for r in reps]}))
else:
    st = pkg.State(n)
    st.apply_circuit(t, fusion_mode=1, tile_qubits=T, tile_jit=1)
    print(json.dumps({"where": "B200", "HHLSV_JIT": os.environ.get("HHLSV_JIT"), "max_err": float(np.abs(st.read() - ref).max())}))
'''

mode = sys.argv[1] if len(sys.argv) > 1 else "cpu"
base = "minb=32,cw=0"
runs = [base] if mode == "cpu" else [base, base + ",ptxas=-O1", "(product default)"]
for cfg in runs:
    env = dict(os.environ)
    if cfg != "(product default)":
        env["HHLSV_JIT"] = cfg
    d = tempfile.mkdtemp()
    env["HHLSV_EMU_DIR"] = d
    env["HHLSV_JIT_DUMP"] = d
    r = subprocess.run([sys.executable, "-c", CASE, ROOT, mode], capture_output=True, text=True, env=env, timeout=900)
    print(r.stdout.strip() or r.stderr[-2000:])
    if mode == "cpu":
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")]
        for c in cub:
            u = subprocess.run(["cuobjdump", "-res-usage", os.path.join(d, c)], capture_output=True, text=True).stdout
            print("  " + " ".join(x for x in u.split() if x.startswith(("REG:", "STACK:"))))
