"""Thin ctypes binding of include/sv.h (argument marshalling only).

Every function here forwards to the same-named C entry point of libhhlsv.so; all
state-vector work happens in the library's CUDA kernels. There is no CPU fallback:
if the library is missing, or no CUDA device is present, calls raise SVError.
PyTorch is used only to hand the library the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhhlsv.so")

SV_DENSE, SV_CONTROLLED, SV_DIAGONAL, SV_RECIP_RY, SV_SWAP = range(5)
_KINDS = {"dense": SV_DENSE, "controlled": SV_CONTROLLED, "diagonal": SV_DIAGONAL, "recip_ry": SV_RECIP_RY,
          "swap": SV_SWAP}
STATUS = ["SV_OK", "SV_E_ARG", "SV_E_RANGE", "SV_E_NOTUNITARY", "SV_E_NOTHERMITIAN", "SV_E_CLOCK",
          "SV_E_ZEROPROB", "SV_E_OOM", "SV_E_CUDA", "SV_E_NCCL"]


class SVError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS[code] if 0 <= code < len(STATUS) else code}: {msg}")
        self.code = code
        self.status = STATUS[code] if 0 <= code < len(STATUS) else str(code)


class sv_dist(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int), ("rank", ctypes.c_int), ("device", ctypes.c_int),
                ("nccl_id", ctypes.c_char_p)]


class sv_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("n_targets", ctypes.c_int), ("targets", ctypes.POINTER(ctypes.c_int)),
                ("n_controls", ctypes.c_int), ("controls", ctypes.POINTER(ctypes.c_int)),
                ("control_values", ctypes.c_uint64), ("data", ctypes.POINTER(ctypes.c_double)),
                ("recip_delta", ctypes.c_double), ("recip_signed", ctypes.c_int), ("recip_snap", ctypes.c_double)]


class sv_fuse_options(ctypes.Structure):
    _fields_ = [("fusion_kmax", ctypes.c_int), ("diag_kmax", ctypes.c_int), ("tile_qubits", ctypes.c_int),
                ("tile_jit", ctypes.c_int), ("fusion_mode", ctypes.c_int)]


class sv_plan_report(ctypes.Structure):
    _fields_ = [("n_logical", ctypes.c_uint64), ("n_fused", ctypes.c_uint64), ("n_passes", ctypes.c_uint64),
                ("alg_bytes", ctypes.c_double), ("pass_bytes", ctypes.c_double)]


class hhl_options(ctypes.Structure):
    _fields_ = [("clock_qubits", ctypes.c_int), ("fusion_kmax", ctypes.c_int), ("tile_qubits", ctypes.c_int),
                ("recip_snap", ctypes.c_double), ("init_fold", ctypes.c_int), ("tile_jit", ctypes.c_int),
                ("diag_kmax", ctypes.c_int), ("qpe_mode", ctypes.c_int),
                ("eig_lambda", ctypes.POINTER(ctypes.c_double)), ("eig_vectors", ctypes.POINTER(ctypes.c_double)),
                ("fusion_mode", ctypes.c_int), ("fused_marginal", ctypes.c_int)]


class hhl_report(ctypes.Structure):
    _fields_ = [("p_success", ctypes.c_double), ("norm2", ctypes.c_double), ("lambda_min", ctypes.c_double),
                ("lambda_max", ctypes.c_double), ("kappa", ctypes.c_double), ("delta", ctypes.c_double),
                ("t_evol", ctypes.c_double), ("n_data", ctypes.c_int), ("n_clock", ctypes.c_int),
                ("n_total", ctypes.c_int), ("n_logical", ctypes.c_uint64), ("n_fused", ctypes.c_uint64),
                ("n_passes", ctypes.c_uint64), ("alg_bytes", ctypes.c_double), ("pass_bytes", ctypes.c_double),
                ("t_frontend_s", ctypes.c_double), ("t_sim_s", ctypes.c_double), ("h2d_bytes", ctypes.c_double),
                ("d2h_bytes", ctypes.c_double), ("x_offset", ctypes.c_int), ("n_orig", ctypes.c_int),
                ("b_norm", ctypes.c_double), ("p_anc1", ctypes.c_double), ("fusion_kmax_used", ctypes.c_int),
                ("model_ms", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["sv_last_error", "sv_version", "sv_nccl_unique_id", "sv_comm_bench", "sv_create", "sv_destroy", "sv_trim_memory",
           "sv_reset", "sv_info", "sv_dump", "sv_restore",
           "sv_qubit_map", "sv_sync", "sv_read", "sv_write", "sv_apply_fused", "sv_apply_circuit",
           "sv_program_create", "sv_program_run", "sv_program_destroy", "sv_program_dump",
           "sv_program_set_timing", "sv_program_timings", "sv_program_stats", "sv_program_marginal", "sv_schedule_dump", "sv_probabilities",
           "sv_norm2", "sv_postselect_slice", "sv_sample", "hhl_plan_size", "hhl_build_program", "hhl_readout", "hhl_solve",
           "hhl_schedule_dump"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libhhlsv.so (raises if it is missing: the product has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise SVError(8, f"{path} not built (run python -m paper_2402_08136_b200.build)")
    L = ctypes.CDLL(path)
    P, c_int, c_u64, c_dbl, vp = ctypes.POINTER, ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
    L.sv_last_error.restype = ctypes.c_char_p
    L.sv_version.restype = ctypes.c_char_p
    sig = {
        "sv_nccl_unique_id": [ctypes.c_char_p],
        "sv_comm_bench": [c_int, c_int, c_int, ctypes.c_char_p, c_int, c_u64, c_int, P(c_dbl), P(c_dbl), P(c_u64)],
        "sv_create": [c_int, P(sv_dist), vp, P(vp)],
        "sv_destroy": [vp], "sv_reset": [vp], "sv_trim_memory": [c_int],
        "sv_info": [vp, P(c_int), P(c_u64), P(vp)],
        "sv_qubit_map": [vp, P(c_int)],
        "sv_sync": [vp],
        "sv_read": [vp, c_u64, c_u64, P(c_dbl)],
        "sv_dump": [vp, ctypes.c_char_p], "sv_restore": [vp, ctypes.c_char_p],
        "sv_write": [vp, c_u64, c_u64, P(c_dbl)],
        "sv_apply_fused": [vp, P(sv_gate), ctypes.c_size_t],
        "sv_apply_circuit": [vp, P(sv_gate), ctypes.c_size_t, P(sv_fuse_options), P(sv_plan_report)],
        "sv_program_create": [vp, P(sv_gate), ctypes.c_size_t, P(sv_fuse_options), P(vp), P(sv_plan_report)],
        "sv_program_run": [vp, vp], "sv_program_destroy": [vp],
        "sv_program_dump": [vp, ctypes.c_char_p, ctypes.c_size_t],
        "sv_program_set_timing": [vp, c_int],
        "sv_program_timings": [vp, P(ctypes.c_float), P(c_int), P(c_dbl), P(c_dbl), P(c_int), ctypes.c_size_t,
                               P(ctypes.c_size_t)],
        "sv_program_stats": [vp, P(c_u64), P(c_u64)],
        "sv_program_marginal": [vp, P(c_dbl)],
        "sv_schedule_dump": [c_int, c_int, P(sv_gate), ctypes.c_size_t, P(sv_fuse_options), ctypes.c_char_p,
                             ctypes.c_size_t, P(sv_plan_report)],
        "sv_probabilities": [vp, P(c_int), c_int, P(c_dbl)],
        "sv_norm2": [vp, P(c_dbl)],
        "sv_postselect_slice": [vp, P(c_int), P(c_int), c_int, P(c_dbl), P(c_u64), c_u64, P(c_dbl)],
        "sv_sample": [vp, c_u64, c_u64, P(c_u64)],
        "hhl_plan_size": [P(c_dbl), P(c_dbl), c_int, P(hhl_options), P(c_int), P(c_int), P(c_int)],
        "hhl_schedule_dump": [P(c_dbl), P(c_dbl), c_int, P(hhl_options), c_int, ctypes.c_char_p, ctypes.c_size_t,
                              P(hhl_report)],
        "hhl_build_program": [vp, P(c_dbl), P(c_dbl), c_int, P(hhl_options), P(vp), P(hhl_report)],
        "hhl_readout": [vp, P(hhl_report), c_int, P(c_dbl), P(c_dbl)],
        "hhl_solve": [P(c_dbl), P(c_dbl), c_int, c_int, P(hhl_options), P(sv_dist), vp, P(c_dbl), P(hhl_report)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = c_int
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise SVError(rc, load().sv_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(lst):
    return (ctypes.c_int * max(1, len(lst)))(*[int(x) for x in lst])


def _current_stream():
    try:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:
        pass
    return ctypes.c_void_p(0)


class _GateArray:
    """Marshal a list of gate dicts (workloads/synthetic.py format) into sv_gate[] (keeps buffers alive)."""

    def __init__(self, gates):
        self.keep = []
        self.arr = (sv_gate * max(1, len(gates)))()
        for i, g in enumerate(gates):
            s = self.arr[i]
            s.kind = _KINDS[g["kind"]]
            t = _ip(g["targets"])
            s.n_targets = len(g["targets"])
            s.targets = t
            c = list(g.get("controls", []))
            ca = _ip(c)
            s.n_controls = len(c)
            s.controls = ca
            s.control_values = int(g.get("cvals", (1 << len(c)) - 1 if c else 0))
            self.keep += [t, ca]
            if "data" in g and g["data"] is not None:
                d = np.ascontiguousarray(np.asarray(g["data"], dtype=np.complex128)).view(np.float64)
                self.keep.append(d)
                s.data = _dp(d)
            s.recip_delta = float(g.get("delta", 0.0))
            s.recip_signed = int(g.get("signed", 1))
            s.recip_snap = float(g.get("snap", 0.0))
        self.n = len(gates)


def _fuse_opts(fusion_kmax=0, diag_kmax=0, tile_qubits=0, tile_jit=0, fusion_mode=0):
    return sv_fuse_options(int(fusion_kmax), int(diag_kmax), int(tile_qubits), int(tile_jit), int(fusion_mode))


def trim_memory(device: int = -1):
    """sv_trim_memory: release the device memory the library's pool caches for reuse."""
    _check(load().sv_trim_memory(int(device)))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().sv_nccl_unique_id(buf))
    return buf.raw


def comm_bench(world: int = 1, rank: int = 0, device: int = -1, nccl_id: bytes | None = None, pattern: int = 0,
               nbytes: int = 1 << 30, reps: int = 5) -> dict:
    """sv_comm_bench: the exchange transport between `world` ranks (pattern 0 pairwise, 1 all-to-all;
    world 1 exchanges with itself). Returns ms per exchange, GB/s sent by this rank, mismatching doubles."""
    if nccl_id is None:
        if world != 1:
            raise SVError(1, "nccl_id required for world > 1")
        nccl_id = nccl_unique_id()
    ms, gbs, bad = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    _check(load().sv_comm_bench(int(world), int(rank), int(device), nccl_id, int(pattern), int(nbytes), int(reps),
                                ctypes.byref(ms), ctypes.byref(gbs), ctypes.byref(bad)))
    return {"ms": ms.value, "gbs": gbs.value, "mismatches": bad.value, "bytes": int(nbytes), "pattern": int(pattern),
            "world": int(world)}


class State:
    """A (sharded) n-qubit state vector on the GPU (sv_create / sv_destroy)."""

    def __init__(self, n_qubits: int, world: int = 1, rank: int = 0, device: int = -1, nccl_id: bytes | None = None,
                 stream=None):
        L = load()
        self._h = ctypes.c_void_p()
        self._dist = None
        if world > 1 or device >= 0:
            self._idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
            self._dist = sv_dist(world, rank, device, ctypes.cast(self._idbuf, ctypes.c_char_p) if self._idbuf else None)
        self.stream = stream if stream is not None else _current_stream()
        _check(L.sv_create(int(n_qubits), ctypes.byref(self._dist) if self._dist else None, self.stream,
                           ctypes.byref(self._h)))
        self.n = int(n_qubits)
        self.world, self.rank = world, rank

    @property
    def handle(self):
        return self._h

    def destroy(self):
        if self._h:
            _check(load().sv_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def reset(self):
        _check(load().sv_reset(self._h))

    def info(self):
        n, la, p = ctypes.c_int(), ctypes.c_uint64(), ctypes.c_void_p()
        _check(load().sv_info(self._h, ctypes.byref(n), ctypes.byref(la), ctypes.byref(p)))
        return n.value, la.value, p.value

    def qubit_map(self):
        m = (ctypes.c_int * self.n)()
        _check(load().sv_qubit_map(self._h, m))
        return list(m)

    def sync(self):
        _check(load().sv_sync(self._h))

    def read(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = (1 << self.n) - first if count is None else count
        out = np.empty(count, dtype=np.complex128)
        _check(load().sv_read(self._h, first, count, _dp(out.view(np.float64))))
        return out

    def dump(self, path: str):
        """sv_dump: checkpoint the state (uint64 length + interleaved re/im doubles, logical order)."""
        _check(load().sv_dump(self._h, os.fsencode(path)))

    def restore(self, path: str):
        """sv_restore: load a checkpoint written by dump() into this state."""
        _check(load().sv_restore(self._h, os.fsencode(path)))

    def write(self, amps, first: int = 0):
        a = np.ascontiguousarray(np.asarray(amps, dtype=np.complex128))
        _check(load().sv_write(self._h, first, a.size, _dp(a.view(np.float64))))

    def apply_fused(self, gates):
        ga = _GateArray(gates)
        _check(load().sv_apply_fused(self._h, ga.arr, ga.n))

    def apply_circuit(self, gates, fusion_kmax=4, diag_kmax=0, tile_qubits=0, tile_jit=0, fusion_mode=0) -> dict:
        ga = _GateArray(gates)
        o = _fuse_opts(fusion_kmax, diag_kmax, tile_qubits, tile_jit, fusion_mode)
        rep = sv_plan_report()
        _check(load().sv_apply_circuit(self._h, ga.arr, ga.n, ctypes.byref(o), ctypes.byref(rep)))
        return {f: getattr(rep, f) for f, _ in rep._fields_}

    def probabilities(self, qubits) -> np.ndarray:
        out = np.empty(1 << len(qubits))
        _check(load().sv_probabilities(self._h, _ip(qubits), len(qubits), _dp(out)))
        return out

    def norm2(self) -> float:
        v = ctypes.c_double()
        _check(load().sv_norm2(self._h, ctypes.byref(v)))
        return v.value

    def postselect_slice(self, fixed_q, fixed_v):
        nfree = self.n - len(fixed_q)
        amps = np.empty(1 << nfree, dtype=np.complex128)
        idx = np.empty(1 << nfree, dtype=np.uint64)
        p = ctypes.c_double()
        _check(load().sv_postselect_slice(self._h, _ip(fixed_q), _ip(fixed_v), len(fixed_q),
                                          _dp(amps.view(np.float64)),
                                          idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), amps.size,
                                          ctypes.byref(p)))
        return amps, idx, p.value

    def sample(self, shots: int, seed: int = 0) -> np.ndarray:
        """sv_sample: `shots` logical basis indices drawn from |a|^2 (deterministic in seed)."""
        out = np.empty(max(1, int(shots)), dtype=np.uint64)
        _check(load().sv_sample(self._h, int(shots), int(seed) & ((1 << 64) - 1),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        return out[:int(shots)]


class Program:
    """A fused, scheduled circuit resident on the device (sv_program_*)."""

    def __init__(self, state: State, handle, report: dict):
        self.state = state
        self._h = handle
        self.report = report

    @classmethod
    def create(cls, state: State, gates, fusion_kmax=4, diag_kmax=0, tile_qubits=0, tile_jit=0, fusion_mode=0):
        ga = _GateArray(gates)
        o = _fuse_opts(fusion_kmax, diag_kmax, tile_qubits, tile_jit, fusion_mode)
        h = ctypes.c_void_p()
        rep = sv_plan_report()
        _check(load().sv_program_create(state.handle, ga.arr, ga.n, ctypes.byref(o), ctypes.byref(h),
                                        ctypes.byref(rep)))
        return cls(state, h, {f: getattr(rep, f) for f, _ in rep._fields_})

    def run(self):
        _check(load().sv_program_run(self.state.handle, self._h))

    def dump(self) -> str:
        buf = ctypes.create_string_buffer(1 << 20)
        _check(load().sv_program_dump(self._h, buf, len(buf)))
        return buf.value.decode()

    def set_timing(self, enable: bool = True):
        _check(load().sv_program_set_timing(self._h, int(enable)))

    def timings(self, with_flops: bool = False):
        """Per-step (ms, kind, bytes, launches[, flops]) of the last run (needs set_timing(True) before it)."""
        n = ctypes.c_size_t()
        _check(load().sv_program_timings(self._h, None, None, None, None, None, 0, ctypes.byref(n)))
        cap = n.value
        ms = (ctypes.c_float * max(1, cap))()
        kd = (ctypes.c_int * max(1, cap))()
        by = (ctypes.c_double * max(1, cap))()
        fl = (ctypes.c_double * max(1, cap))()
        la = (ctypes.c_int * max(1, cap))()
        _check(load().sv_program_timings(self._h, ms, kd, by, fl, la, cap, ctypes.byref(n)))
        if with_flops:
            return [(ms[i], kd[i], by[i], la[i], fl[i]) for i in range(cap)]
        return [(ms[i], kd[i], by[i], la[i]) for i in range(cap)]

    def stats(self):
        la, h2d = ctypes.c_uint64(), ctypes.c_uint64()
        _check(load().sv_program_stats(self._h, ctypes.byref(la), ctypes.byref(h2d)))
        return {"launches": la.value, "h2d_bytes": h2d.value}

    def marginal(self):
        """(P(ancilla = 0), P(ancilla = 1)) of the last run, accumulated by the program's last tile pass
        (single-GPU HHL programs; raises SVError otherwise)."""
        out = (ctypes.c_double * 2)()
        _check(load().sv_program_marginal(self._h, out))
        return out[0], out[1]

    def destroy(self):
        if self._h:
            _check(load().sv_program_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


STEP_KINDS = ["init_zero", "init_product", "dense", "diagonal", "recip_ry", "tile", "exchange"]


def schedule_dump(n_qubits: int, gates, world: int = 1, fusion_kmax=4, diag_kmax=0, tile_qubits=0, tile_jit=0,
                  fusion_mode=0):
    """Host-only: fuse + schedule a logical gate list (no GPU needed). Returns (text, report).
    tile_jit=1 also generates and NVRTC-compiles (sm_100a) every tile pass."""
    ga = _GateArray(gates)
    o = _fuse_opts(fusion_kmax, diag_kmax, tile_qubits, tile_jit, fusion_mode)
    buf = ctypes.create_string_buffer(1 << 22)
    rep = sv_plan_report()
    _check(load().sv_schedule_dump(int(n_qubits), int(world), ga.arr, ga.n, ctypes.byref(o), buf, len(buf),
                                   ctypes.byref(rep)))
    return buf.value.decode(), {f: getattr(rep, f) for f, _ in rep._fields_}


class _Opts:
    """hhl_options plus the buffers its eig_* pointers reference (kept alive with it)."""

    def __init__(self, clock_qubits=0, fusion_kmax=0, tile_qubits=0, recip_snap=1e-5, init_fold=0, tile_jit=0,
                 diag_kmax=0, qpe_mode=0, eig=None, fusion_mode=0, fused_marginal=0):
        self.o = hhl_options(int(clock_qubits), int(fusion_kmax), int(tile_qubits), float(recip_snap),
                             int(init_fold), int(tile_jit), int(diag_kmax), int(qpe_mode))
        self.o.fusion_mode = int(fusion_mode)
        self.o.fused_marginal = int(fused_marginal)
        if eig is not None:          # (lambda, V): caller-supplied eigendecomposition of the padded A
            self.lam = np.ascontiguousarray(eig[0], dtype=np.float64)
            self.V = np.ascontiguousarray(eig[1], dtype=np.float64)
            if self.V.shape != (self.lam.size, self.lam.size):
                raise SVError(1, "eig: V must be N x N with N = len(lambda)")
            self.o.eig_lambda = _dp(self.lam)
            self.o.eig_vectors = _dp(self.V)

    def ref(self):
        return ctypes.byref(self.o)


def _opts(**kw):
    return _Opts(**kw)


def hhl_plan_size(A, b, **kw):
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    o = _opts(**kw)
    nd, nc, nt = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(load().hhl_plan_size(_dp(A), _dp(b), b.size, o.ref(), ctypes.byref(nd), ctypes.byref(nc),
                                ctypes.byref(nt)))
    return nd.value, nc.value, nt.value


def hhl_schedule_dump(A, b, world: int = 1, **kw):
    """Host-only: the schedule hhl_build_program would run for (A, b) on `world` ranks.
    Returns (text, report dict)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    o = _opts(**kw)
    buf = ctypes.create_string_buffer(1 << 22)
    rep = hhl_report()
    _check(load().hhl_schedule_dump(_dp(A), _dp(b), b.size, o.ref(), int(world), buf, len(buf),
                                    ctypes.byref(rep)))
    return buf.value.decode(), {f: getattr(rep, f) for f, _ in rep._fields_}


class HHLProgram(Program):
    """hhl_build_program: the HHL circuit for (A, b) as a resident program on `state`."""

    @classmethod
    def build(cls, state: State, A, b, **kw):
        A = np.ascontiguousarray(A, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        o = _opts(**kw)
        h = ctypes.c_void_p()
        rep = hhl_report()
        _check(load().hhl_build_program(state.handle, _dp(A), _dp(b), b.size, o.ref(), ctypes.byref(h),
                                        ctypes.byref(rep)))
        p = cls(state, h, rep.as_dict())
        p._rep = rep
        return p

    def readout(self):
        x = np.empty(self._rep.n_orig)
        ps = ctypes.c_double()
        _check(load().hhl_readout(self.state.handle, ctypes.byref(self._rep), self._rep.n_orig, _dp(x),
                                  ctypes.byref(ps)))
        return x, ps.value


def hhl_solve(A, b, clock_qubits=0, world=1, rank=0, device=-1, nccl_id=None, stream=None, **kw):
    """Solve A x = b with the simulated HHL circuit on the GPU(s). A, b, x are host arrays."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    o = _opts(clock_qubits=clock_qubits, **kw)
    x = np.empty(b.size)
    rep = hhl_report()
    dist = None
    idbuf = None
    if world > 1 or device >= 0:
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        dist = sv_dist(world, rank, device, ctypes.cast(idbuf, ctypes.c_char_p) if idbuf else None)
    _check(load().hhl_solve(_dp(A), _dp(b), b.size, int(clock_qubits), o.ref(),
                            ctypes.byref(dist) if dist else None, stream if stream is not None else _current_stream(),
                            _dp(x), ctypes.byref(rep)))
    return x, rep.as_dict()
