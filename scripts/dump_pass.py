"""Print the schedule (ops per tile) of the S30 HHL program (developer tool, GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08136_b200 as pkg  # noqa: E402
from workloads import configs  # noqa: E402
A, b, nc = configs.get(os.environ.get("CFG", "S30"))
st = pkg.State(configs.n_qubits(os.environ.get("CFG", "S30")))
prog = pkg.HHLProgram.build(st, A, b, clock_qubits=nc, fusion_kmax=1, tile_qubits=11, qpe_mode=1, tile_jit=1)
print(prog.dump())
