"""CPU oracle wall time on the full Table 1 / small configs, on the host it runs on:
all hardware threads and one thread, with the CPU model. One JSON object (default
profiles/r02_oracle_timing.json when run with --write).

    python scripts/oracle_timing.py [--write]
The oracle is oracle/sv_oracle.c (OpenMP) applying the UNFUSED logical HHL list (oracle/hhl.py build)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, time
sys.path.insert(0, sys.argv[1])
from oracle import hhl as ohhl, sim
from workloads import configs
out = {}
for name in ("C1", "C2", "C3p", "C3", "B30", "S20"):
    A, b, nc = configs.get(name)
    p = ohhl.plan(A, b, nc)
    g = ohhl.build(p)
    sim.run(g[:4], p.n)                         # warm-up (library load, OpenMP pool)
    best = 1e30
    for _ in range(3):
        t = time.perf_counter()
        sim.run(g, p.n)
        best = min(best, time.perf_counter() - t)
    out[name] = {"n_qubits": p.n, "logical_gates": len(g), "seconds": best, "threads": sim.n_threads()}
print(json.dumps(out))
'''


def run(threads):
    env = dict(os.environ)
    if threads:
        env["OMP_NUM_THREADS"] = str(threads)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, env=env, timeout=1800)
    if r.returncode:
        raise SystemExit(r.stderr)
    return json.loads(r.stdout)


model = "unknown"
try:
    model = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
except Exception:
    pass
res = {"host_cpu": model, "host_threads": os.cpu_count(), "all_threads": run(None), "one_thread": run(1),
       "how": "best of 3 full oracle runs of the unfused logical HHL list (oracle/sv_oracle.c, OpenMP), per config"}
print(json.dumps(res, indent=1))
if "--write" in sys.argv:
    with open(os.path.join(ROOT, "profiles", "r02_oracle_timing.json"), "w") as f:
        json.dump(res, f, indent=1)
