"""Host emulation of the generated NVRTC tile passes with race / bounds / barrier checking.

compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing a reset), so the
generated CUDA source is checked on the CPU instead:

* the library's host-only planner (hhl_schedule_dump / sv_schedule_dump with tile_jit = 1 and
  HHLSV_EMU_DIR set) lowers the program exactly as on the GPU and exports every pass: its CUDA
  source (without the device prelude), the data blob, the by-value kernel-parameter values and the
  launch parameters;
* each pass source is compiled as host C++20 against HOST_PRELUDE below (the device prelude's
  functions re-implemented with checks) with AddressSanitizer, and run as CUDA would: one std::thread
  per CUDA thread of a CTA, a std::barrier for bar.sync, several persistent CTAs one after another;
* racecheck: every shared-memory access is recorded per 8-byte word with the accessing thread and its
  barrier epoch; a read of a word another thread wrote in the same epoch (RAW), or a write of a word
  another thread read or wrote in the same epoch (WAR / WAW), is a race;
* memcheck: shared accesses outside the launch's dynamic shared memory, global reads / writes outside
  the state or the blob (ASan also guards the heap buffers); every state amplitude written at most once
  per pass;
* synccheck: every thread of a CTA passes the same number of barriers.
The emulated program's final state is compared with the oracle by the tests (tests/test_jit_emulation.py).
"""
from __future__ import annotations

import hashlib
import os
import re
import subprocess
import tempfile

import numpy as np

HOST_PRELUDE = r'''
#include <atomic>
#include <barrier>
#include <memory>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sys/mman.h>
#include <thread>
#include <unordered_set>
#include <vector>
typedef unsigned long long u64;
typedef unsigned int u32;
struct double2 { double x, y; };
struct Dim { unsigned x = 0, y = 0, z = 0; };
static thread_local Dim threadIdx;
static Dim blockIdx, gridDim;
static thread_local int g_tid = 0, g_epoch = 0, g_bars = 0;
// warp-synchronous ordering (mma.sync): accesses of two lanes of one warp separated by a warp-collective
// MMA are ordered even inside one barrier epoch; g_wsync counts the MMAs a thread passed
static thread_local int g_wsync = 0;
static std::barrier<> *g_bar = nullptr;
static unsigned char *g_smem = nullptr;
static size_t g_smem_bytes = 0;
static const double2 *g_psi = nullptr, *g_blob = nullptr;
static size_t g_psi_n = 0, g_blob_n = 0;
static std::unordered_set<u64> g_written;
// per 8-byte word: last write (epoch, thread, warp-sync count) and the reads of the current epoch
// (one reader's thread or -2, the readers' warp or -3 when several warps, the largest warp-sync count)
struct Shadow { int we = -1, wt = -1, wws = -1, re = -1, rt = -1, rwarp = -1, rws = -1; };
static std::vector<Shadow> g_sh;
static std::mutex g_mu;
static std::atomic<long> g_races{0}, g_oob{0}, g_double{0};
#define __device__
#define __forceinline__ inline
static void report(const char *what, unsigned long long a) {
    if (g_races + g_oob + g_double < 40) fprintf(stderr, "%s at %llu (tid %d, epoch %d, cta %u)\n", what, a, g_tid, g_epoch, blockIdx.x);
}
static void sm_access(u32 a, unsigned bytes, bool write) {
    if ((size_t)a + bytes > g_smem_bytes) { g_oob++; report("SMEM_OOB", a); return; }
    std::lock_guard<std::mutex> lk(g_mu);
    for (u32 w = a / 8; w < (a + bytes + 7) / 8; w++) {
        Shadow &s = g_sh[w];
        const int warp = g_tid >> 5;
        if (s.we == g_epoch && s.wt != g_tid && !((s.wt >> 5) == warp && s.wws < g_wsync)) {
            g_races++;
            report(write ? "RACE_WAW" : "RACE_RAW", w * 8ull);
        }
        if (write) {
            if (s.re == g_epoch && s.rt != g_tid && !(s.rwarp == warp && s.rws < g_wsync)) {
                g_races++;
                report("RACE_WAR", w * 8ull);
            }
            s.we = g_epoch; s.wt = g_tid; s.wws = g_wsync;
        } else {
            if (s.re != g_epoch) { s.re = g_epoch; s.rt = g_tid; s.rwarp = warp; s.rws = g_wsync; }
            else {
                if (s.rt != g_tid) s.rt = -2;      // several readers this epoch
                if (s.rwarp != warp) s.rwarp = -3;
                if (g_wsync > s.rws) s.rws = g_wsync;
            }
        }
    }
}
static bool in_psi(const void *p, size_t bytes) {
    const char *c = (const char *)p, *b = (const char *)g_psi;
    return c >= b && c + bytes <= b + g_psi_n * sizeof(double2);
}
static bool in_blob(const void *p, size_t bytes) {
    const char *c = (const char *)p, *b = (const char *)g_blob;
    return c >= b && c + bytes <= b + g_blob_n * sizeof(double2);
}
__device__ __forceinline__ u32 swz(u32 u) { return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u); }
__device__ __forceinline__ u64 insz(u64 x, int p) { return ((x >> p) << (p + 1)) | (x & ((1ull << p) - 1ull)); }
static inline u64 __cvta_generic_to_shared(const void *) { return 0; }
static inline double2 lds(u32 a) { sm_access(a, 16, false); double2 v; memcpy(&v, g_smem + a, 16); return v; }
static inline void sts(u32 a, double2 v) { sm_access(a, 16, true); memcpy(g_smem + a, &v, 16); }
static inline u64 lds64(u32 a) { sm_access(a, 8, false); u64 v; memcpy(&v, g_smem + a, 8); return v; }
static inline void sts64(u32 a, u64 v) { sm_access(a, 8, true); memcpy(g_smem + a, &v, 8); }
static inline void stsd(u32 a, double v) { sm_access(a, 8, true); memcpy(g_smem + a, &v, 8); }
static inline double ldsd(u32 a) { sm_access(a, 8, false); double v; memcpy(&v, g_smem + a, 8); return v; }
static inline void cp_async16s(u32 s, const void *g) {
    if (!in_psi(g, 16)) { g_oob++; report("GLOBAL_READ_OOB(cp.async)", (unsigned long long)g); return; }
    sm_access(s, 16, true); memcpy(g_smem + s, g, 16);
}
static inline void cp_async_commit() {}
static inline void cp_async_wait0() {}
static inline void cp_async_wait1() {}
static inline double2 ldcs_v(const double2 *g) {
    if (!in_psi(g, 16)) { g_oob++; report("GLOBAL_READ_OOB", (unsigned long long)(g - g_psi)); return double2{0, 0}; }
    return *g;
}
static inline void bar() { g_bar->arrive_and_wait(); g_epoch++; g_bars++; }
static inline void pf_l2(const void *g) {
    if (!in_psi(g, 1)) { g_oob++; report("PREFETCH_OOB", (unsigned long long)g); }
}
static inline void gstore(double2 *p, double2 v) {
    if (!in_psi(p, 16)) { g_oob++; report("GLOBAL_WRITE_OOB", (unsigned long long)(p - g_psi)); return; }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_written.insert((u64)(p - g_psi)).second) { g_double++; report("DOUBLE_WRITE", (unsigned long long)(p - g_psi)); }
    }
    *p = v;
}
static inline void __stcs(double2 *p, double2 v) { gstore(p, v); }
template <class T> static inline T __ldg(const T *p) {
    if (!in_blob(p, sizeof(T))) { g_oob++; report("BLOB_READ_OOB", (unsigned long long)p); return T{}; }
    return *p;
}
struct SRef {
    u32 a;
    operator double2() const { return lds(a); }
    void operator=(double2 v) const { sts(a, v); }
    void operator=(const SRef &o) const { sts(a, lds(o.a)); }
};
struct SArr {
    u32 b;
    SRef operator[](u32 i) const { return SRef{b + (i << 4)}; }
    SArr operator+(u32 o) const { return SArr{b + (o << 4)}; }
    u32 at(u32 i) const { return b + (i << 4); }
};
struct SRef64 {
    u32 a;
    operator u64() const { return lds64(a); }
    void operator=(u64 v) const { sts64(a, v); }
};
struct SArr64 {
    u32 b;
    SRef64 operator[](u32 i) const { return SRef64{b + (i << 3)}; }
};
static inline double2 mk(double x, double y) { double2 r; r.x = x; r.y = y; return r; }
static inline double2 cmul(const double2 a, const double2 b) { return mk(std::fma(a.x, b.x, -a.y * b.y), std::fma(a.x, b.y, a.y * b.x)); }
// mma.sync.m8n8k4.f64 as a warp collective: lane l holds A[l / 4][l % 4], B[l % 4][l / 4] and
// D[l / 4][2 (l % 4) + {0, 1}] (PTX fragment layouts)
static std::vector<std::unique_ptr<std::barrier<>>> g_wbars;
static double g_wa[64][32], g_wb[64][32];
static inline void dmma884(double &d0, double &d1, double a, double b) {
    const int w = g_tid >> 5, l = g_tid & 31;
    g_wa[w][l] = a; g_wb[w][l] = b;
    g_wbars[w]->arrive_and_wait();
    g_wsync++;
    const int row = l >> 2, c0 = 2 * (l & 3);
    for (int q = 0; q < 4; q++) {
        d0 = std::fma(g_wa[w][row * 4 + q], g_wb[w][c0 * 4 + q], d0);
        d1 = std::fma(g_wa[w][row * 4 + q], g_wb[w][(c0 + 1) * 4 + q], d1);
    }
    g_wbars[w]->arrive_and_wait();
}
static inline double __ddiv_rn(double a, double b) { return a / b; }
using std::fma; using std::sqrt; using std::fabs;
static inline double recip_s(u64 m, int n_c, double dL, int sg, double snap) {
    if (m == 0) return 0.0;
    double sign = 1.0;
    u64 mp = m;
    if (sg && m >= (1ull << (n_c - 1))) { mp = (1ull << n_c) - m; sign = -1.0; }
    const double r = __ddiv_rn(dL, (double)mp);
    const double s = fabs(r - 1.0) <= snap ? 1.0 : (r < 1.0 ? r : 0.0);
    return sign * s;
}
'''

MAIN = r'''
static std::vector<char> slurp(const char *path) {
    FILE *f = fopen(path, "rb");
    if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
    fseek(f, 0, SEEK_END); long n = ftell(f); fseek(f, 0, SEEK_SET);
    std::vector<char> v(n);
    if (n && fread(v.data(), 1, n, f) != (size_t)n) { fprintf(stderr, "short read %s\n", path); exit(2); }
    fclose(f);
    return v;
}
int main(int argc, char **argv) {
    // psi_in psi_out blob cw n_tiles rank_base nthr smem_bytes n_cta [n_amps]
    // psi_in "-": a zero state of n_amps amplitudes mapped lazily (full-size passes, checks only)
    std::vector<char> blob_b = slurp(argv[3]), cw_b = slurp(argv[4]);
    const u64 n_tiles = strtoull(argv[5], 0, 10), rank_base = strtoull(argv[6], 0, 10);
    const int nthr = atoi(argv[7]);
    g_smem_bytes = (size_t)atoll(argv[8]);
    const unsigned ncta = (unsigned)atoi(argv[9]);
    const bool lazy = strcmp(argv[1], "-") == 0;
    std::vector<double> red_b(2 * ncta + 2, std::nan(""));   // fused-marginal partials (passes with red)
    double2 *psi;
    if (lazy) {
        g_psi_n = strtoull(argv[10], 0, 10);
        psi = (double2 *)mmap(nullptr, g_psi_n * 16, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
        if (psi == MAP_FAILED) { fprintf(stderr, "mmap failed\n"); return 2; }
    } else {
        std::vector<char> psi_b = slurp(argv[1]);
        psi = (double2 *)malloc(psi_b.size());
        memcpy(psi, psi_b.data(), psi_b.size());
        g_psi_n = psi_b.size() / 16;
    }
    double2 *blob = (double2 *)malloc(blob_b.size() + 16);
    memcpy(blob, blob_b.data(), blob_b.size());
    g_psi = psi; g_blob = blob; g_blob_n = blob_b.size() / 16;
    g_smem = (unsigned char *)malloc(g_smem_bytes);
    g_sh.assign(g_smem_bytes / 8 + 2, Shadow{});
    gridDim.x = ncta;
    std::vector<int> bars(nthr);
    long sync_err = 0;
    for (unsigned c = 0; c < ncta; c++) {
        blockIdx.x = c;
        memset(g_smem, 0xA5, g_smem_bytes);        // stale data: an uninitialised read shows up in the result
        std::fill(g_sh.begin(), g_sh.end(), Shadow{});
        std::barrier<> br(nthr);
        g_bar = &br;
        g_wbars.clear();
        for (int w = 0; w * 32 < nthr; w++) g_wbars.emplace_back(new std::barrier<>(std::min(32, nthr - 32 * w)));
        std::vector<std::thread> th;
        for (int t = 0; t < nthr; t++)
            th.emplace_back([&, t] {
                threadIdx.x = (unsigned)t; g_tid = t; g_epoch = 0; g_bars = 0; g_wsync = 0;
                KERNEL_CALL;
                bars[t] = g_bars;
                br.arrive_and_drop();
            });
        for (auto &x : th) x.join();
        for (int t = 1; t < nthr; t++) if (bars[t] != bars[0]) sync_err++;
    }
    if (!lazy) { FILE *f = fopen(argv[2], "wb"); fwrite(psi, 16, g_psi_n, f); fclose(f); }
    printf("races %ld oob %ld double_writes %ld sync_mismatch %ld barriers %d\n", (long)g_races, (long)g_oob,
           (long)g_double, sync_err, bars[0]);
    if (HAS_RED) {      // the CTA partials in launch order (the device sums them the same way)
        double s0 = 0.0, s1 = 0.0;
        for (unsigned c = 0; c < ncta; c++) { s0 += red_b[2 * c]; s1 += red_b[2 * c + 1]; }
        fprintf(stderr, "RED %.17g %.17g\n", s0, s1);
    }
    return 0;
}
'''

_BUILD_DIR = os.path.join(tempfile.gettempdir(), "hhlsv_jit_emu")


def _host_source(src: str) -> tuple[str, bool]:
    """Turn one generated pass (device code after the prelude) into host C++."""
    s = src.replace("extern __shared__ __align__(16) unsigned char smem_raw[];", "unsigned char *smem_raw = g_smem;")
    s = re.sub(r'extern "C" __global__ void __launch_bounds__\(\d+, \d+\) hhlsv_tile', "static void hhlsv_tile", s)
    s = s.replace("double2 *__restrict__ psi", "double2 *psi").replace("const double2 *__restrict__ blob",
                                                                       "const double2 *blob")
    s = s.replace("psi[addr(base, u)] = cur[swz(u)];", "gstore(&psi[addr(base, u)], cur[swz(u)]);")
    s = s.replace("psi[ad] = x;", "gstore(&psi[ad], x);")
    s = s.replace("double *__restrict__ red", "double *red")
    has_cw = "const CWArg cwa" in s
    return s, has_cw


def build_pass(src: str) -> str:
    """Compile one pass source into an emulator executable (cached by content)."""
    os.makedirs(_BUILD_DIR, exist_ok=True)
    body, has_cw = _host_source(src)
    has_red = "double *red" in body
    call = "hhlsv_tile(psi, blob, n_tiles, rank_base, 0ull" + (", red_b.data()" if has_red else "") + (
        ", *(const CWArg *)cw_b.data())" if has_cw else ")")
    full = HOST_PRELUDE + body + MAIN.replace("KERNEL_CALL", call).replace("HAS_RED", "true" if has_red else "false")
    tag = hashlib.sha1(full.encode()).hexdigest()[:16]
    exe = os.path.join(_BUILD_DIR, f"pass_{tag}")
    if not os.path.exists(exe):
        cpp = exe + ".cpp"
        with open(cpp, "w") as f:
            f.write(full)
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-ffp-contract=off", "-fsanitize=address,undefined",
                               "-fno-omit-frame-pointer", "-pthread", cpp, "-o", exe + ".tmp"])
        os.replace(exe + ".tmp", exe)
    return exe


def prebuild(emu_dir: str):
    """Compile every exported pass of a program concurrently (the builds dominate the tests' time)."""
    from concurrent.futures import ThreadPoolExecutor
    with open(os.path.join(emu_dir, "launches.txt")) as f:
        idx = [ln.split()[1] for ln in f if ln.startswith("TILE")]
    srcs = []
    for i in idx:
        with open(os.path.join(emu_dir, f"src_{i}.cu")) as f:
            srcs.append(f.read())
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        list(ex.map(build_pass, srcs))


def check_full_size(emu_dir: str, n_amps: int, tiles: int = 4, max_cta: int = 2):
    """Race / bounds / barrier checks of every exported pass at its real launch size, restricted to the
    first `tiles` tiles (a prefix of the real persistent-loop schedule) on a lazily mapped zero state of
    n_amps amplitudes: the bench's own S30 kernels, without needing 16 GiB of host memory."""
    reports = []
    prebuild(emu_dir)
    with open(os.path.join(emu_dir, "launches.txt")) as f:
        lines = [ln.split() for ln in f if ln.strip()]
    for t in lines:
        if t[0] != "TILE":
            continue
        i, n_tiles, T, rank_base, smem, nthr = t[1], int(t[2]), int(t[3]), int(t[4]), int(t[5]), int(t[6])
        with open(os.path.join(emu_dir, f"src_{i}.cu")) as f:
            exe = build_pass(f.read())
        nt = min(tiles, n_tiles)
        out = subprocess.run([exe, "-", "-", os.path.join(emu_dir, "blob.bin"), os.path.join(emu_dir, f"cw_{i}.bin"),
                              str(nt), str(rank_base), str(nthr), str(smem), str(min(max_cta, nt)), str(n_amps)],
                             capture_output=True, text=True, timeout=900,
                             env=dict(os.environ, ASAN_OPTIONS="detect_leaks=0"))
        if out.returncode != 0:
            raise RuntimeError(f"emulated pass {i} failed ({out.returncode}):\n{out.stderr[-3000:]}")
        vals = dict(zip(out.stdout.split()[0::2], map(int, out.stdout.split()[1::2])))
        vals.update(pass_index=int(i), T=T, tiles=nt, launch_tiles=n_tiles, nthr=nthr, smem=smem)
        reports.append(vals)
    return reports


def run_program(emu_dir: str, psi: np.ndarray, max_cta: int = 3):
    """Run every exported launch of a program on psi (physical order). Returns (psi_out, reports):
    one dict per tile pass with the checker counts. Non-tile launches other than the skipped fused
    init are not supported (the tests choose programs made of tile passes)."""
    psi = np.ascontiguousarray(psi, dtype=np.complex128).copy()
    reports = []
    prebuild(emu_dir)
    with open(os.path.join(emu_dir, "launches.txt")) as f:
        lines = [ln.split() for ln in f if ln.strip()]
    for t in lines:
        if t[0] == "SKIP":
            continue
        if t[0] != "TILE":
            raise RuntimeError(f"launch kind {t[2]} is not emulated")
        i, n_tiles, T, rank_base, smem, nthr = t[1], int(t[2]), int(t[3]), int(t[4]), int(t[5]), int(t[6])
        with open(os.path.join(emu_dir, f"src_{i}.cu")) as f:
            exe = build_pass(f.read())
        pin = os.path.join(emu_dir, f"psi_{i}_in.bin")
        pout = os.path.join(emu_dir, f"psi_{i}_out.bin")
        psi.tofile(pin)
        ncta = max(1, min(max_cta, n_tiles))
        out = subprocess.run([exe, pin, pout, os.path.join(emu_dir, "blob.bin"), os.path.join(emu_dir, f"cw_{i}.bin"),
                              str(n_tiles), str(rank_base), str(nthr), str(smem), str(ncta)],
                             capture_output=True, text=True, timeout=600,
                             env=dict(os.environ, ASAN_OPTIONS="detect_leaks=0"))
        if out.returncode != 0:
            raise RuntimeError(f"emulated pass {i} failed ({out.returncode}):\n{out.stderr[-3000:]}")
        vals = dict(zip(out.stdout.split()[0::2], map(int, out.stdout.split()[1::2])))
        vals.update(T=T, n_tiles=n_tiles, ncta=ncta, log=out.stderr[-2000:])
        for ln in out.stderr.splitlines():
            if ln.startswith("RED "):
                vals["red"] = tuple(float(x) for x in ln.split()[1:3])
        reports.append(vals)
        psi = np.fromfile(pout, dtype=np.complex128)
    return psi, reports


def final_map(dump_text: str):
    for ln in dump_text.splitlines():
        if ln.startswith("FINAL_MAP"):
            return [int(x) for x in ln.split()[1:]]
    return None


def to_logical(psi_phys: np.ndarray, phys_of_logical) -> np.ndarray:
    n = len(phys_of_logical)
    idx = np.arange(1 << n, dtype=np.int64)
    P = np.zeros_like(idx)
    for q, b in enumerate(phys_of_logical):
        P |= ((idx >> q) & 1) << b
    return psi_phys[P]
