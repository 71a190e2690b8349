// Tile-pass specialisation with NVRTC (sm_100a) — DESIGN.md §Tile / §JIT.
//
// The generic k_tile kernel interprets each op descriptor for every tile; at 2^30
// amplitudes that per-op dispatch (dependent shared loads, branches, bit loops) costs
// ~1 ms per op, 4-5x its FP64 work. Every op of a pass is identical for all tiles, so at
// program-creation time we emit one straight-line CUDA kernel per tile pass in which the
// tile bits, register phases, register-slot indices, control masks, bit runs and blob
// offsets are compile-time constants, compile it with NVRTC for sm_100a, and launch it
// through the runtime's library API. Matrix/table VALUES stay in the program's device
// blob, so the generated source depends only on the circuit's structure and is cached
// (in-process, keyed by the exact source text).
#include <dlfcn.h>

#include <algorithm>
#include <charconv>
#include <type_traits>
#include <functional>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <future>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"
#include "jit.h"

namespace hhlsv {

// ------------------------------------------------------------------ NVRTC ----
namespace {
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;
struct Nvrtc {
    void *h = nullptr;
    nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int, const char *const *,
                            const char *const *) = nullptr;
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *) = nullptr;
    nvrtcResult_t (*cubinSize)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*cubin)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*logSize)(nvrtcProgram_t, size_t *) = nullptr;
    nvrtcResult_t (*log)(nvrtcProgram_t, char *) = nullptr;
    nvrtcResult_t (*destroy)(nvrtcProgram_t *) = nullptr;
    const char *(*errStr)(nvrtcResult_t) = nullptr;
    std::string why;
    bool ok = false;
};

Nvrtc &nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {getenv("HHLSV_NVRTC_LIB"), "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                               "libnvrtc.so"};
        for (const char *nm : names) {
            if (!nm) continue;
            n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
            if (n.h) break;
        }
        if (!n.h) {
            n.why = "cannot dlopen libnvrtc.so.12 (set HHLSV_NVRTC_LIB)";
            return;
        }
#define SYM(f, s)                                                   \
    n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.h, s));           \
    if (!n.f) {                                                     \
        n.why = "libnvrtc lacks " s;                                \
        return;                                                     \
    }
        SYM(create, "nvrtcCreateProgram")
        SYM(compile, "nvrtcCompileProgram")
        SYM(cubinSize, "nvrtcGetCUBINSize")
        SYM(cubin, "nvrtcGetCUBIN")
        SYM(logSize, "nvrtcGetProgramLogSize")
        SYM(log, "nvrtcGetProgramLog")
        SYM(destroy, "nvrtcDestroyProgram")
        SYM(errStr, "nvrtcGetErrorString")
#undef SYM
        n.ok = true;
    });
    return n;
}

const char *kPrelude = R"(
typedef unsigned long long u64;
typedef unsigned int u32;
__device__ __forceinline__ u32 swz(u32 u) { return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u); }
__device__ __forceinline__ u64 insz(u64 x, int p) { return ((x >> p) << (p + 1)) | (x & ((1ull << p) - 1ull)); }
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// Shared memory through explicit 32-bit shared-window addresses (nvcc's addressing form; NVRTC's
// default 64-bit shared-pointer arithmetic tripped a ptxas -O2/-O3 miscompilation on some of these
// kernels). Every shared access and barrier is a volatile asm: the compiler keeps their program
// order (volatile asm statements are never reordered with respect to each other); the
// "memory" clobber is added when JitConfig::smem_clobber is set.
#ifdef HHLSV_SMEM_CLOBBER
#define HHLSV_CLB : "memory"
#else
#define HHLSV_CLB
#endif
__device__ __forceinline__ double2 lds(u32 a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) HHLSV_CLB);
    return v;
}
__device__ __forceinline__ void sts(u32 a, double2 v) { asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) HHLSV_CLB); }
__device__ __forceinline__ u64 lds64(u32 a) {
    u64 v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(u32 a, u64 v) { asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v)); }
__device__ __forceinline__ void stsd(u32 a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ double ldsd(u32 a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) HHLSV_CLB);
    return v;
}
// Streaming HBM loads of tile data: not allocated in L1 (an SM must never keep lines another SM
// writes during the pass: a stale line would survive into the next pass), volatile with a memory
// clobber (never moved across this thread's own stores or re-executed by the compiler)
__device__ __forceinline__ double2 ldcs_v(const double2 *g) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(g) : "memory");
    return v;
}
__device__ __forceinline__ void bar() { asm volatile("bar.sync 0;" ::: "memory"); }
__device__ __forceinline__ void pf_l2(const void *g) { asm volatile("prefetch.global.L2 [%0];" ::"l"(g)); }
struct SRef {
    u32 a;
    __device__ __forceinline__ operator double2() const { return lds(a); }
    __device__ __forceinline__ void operator=(double2 v) const { sts(a, v); }
    // element copy (a = b between two slots copies the value, not the proxy)
    __device__ __forceinline__ void operator=(const SRef &o) const { sts(a, lds(o.a)); }
};
struct SArr {      // double2 array in shared memory
    u32 b;
    __device__ __forceinline__ SRef operator[](u32 i) const { return SRef{b + (i << 4)}; }
    __device__ __forceinline__ SArr operator+(u32 o) const { return SArr{b + (o << 4)}; }
    __device__ __forceinline__ u32 at(u32 i) const { return b + (i << 4); }
};
struct SRef64 {
    u32 a;
    __device__ __forceinline__ operator u64() const { return lds64(a); }
    __device__ __forceinline__ void operator=(u64 v) const { sts64(a, v); }
};
struct SArr64 {
    u32 b;
    __device__ __forceinline__ SRef64 operator[](u32 i) const { return SRef64{b + (i << 3)}; }
};
__device__ __forceinline__ void cp_async16s(u32 s, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ double2 mk(double x, double y) { double2 r; r.x = x; r.y = y; return r; }
// FP64 tensor-core MMA, m8n8k4 (warp-collective): {d0, d1} += A (8x4, row) x B (4x8, col)
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 cmul(const double2 a, const double2 b) {
    return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double recip_s(u64 m, int n_c, double dL, int sg, double snap) {
    if (m == 0) return 0.0;
    double sign = 1.0;
    u64 mp = m;
    if (sg && m >= (1ull << (n_c - 1))) { mp = (1ull << n_c) - m; sign = -1.0; }
    const double r = __ddiv_rn(dL, (double)mp);
    const double s = fabs(r - 1.0) <= snap ? 1.0 : (r < 1.0 ? r : 0.0);
    return sign * s;
}
)";

uint32_t swz_host(uint32_t u) { return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u); }

int dep_slot(int c, int M) {   // deposit bits of c into the set bits of M (4-bit register masks)
    int out = 0, bit = 0;
    for (int i = 0; i < 4; i++)
        if ((M >> i) & 1) {
            if ((c >> bit) & 1) out |= 1 << i;
            bit++;
        }
    return out;
}

// Append-only source buffer for the generator (std::ostringstream formatting was ~half of a program's
// host front end): strings and characters appended as is, integers via std::to_chars, doubles as %g
// (the ostringstream defaults), so the generated text is unchanged.
struct SrcBuf {
    std::string s;
    SrcBuf() { s.reserve(1 << 16); }
    SrcBuf &operator<<(const std::string &x) { s += x; return *this; }
    SrcBuf &operator<<(const char *x) { s += x; return *this; }
    SrcBuf &operator<<(char c) { s += c; return *this; }
    SrcBuf &operator<<(signed char c) { s += (char)c; return *this; }
    SrcBuf &operator<<(unsigned char c) { s += (char)c; return *this; }
    SrcBuf &operator<<(bool b) { s += b ? '1' : '0'; return *this; }
    SrcBuf &operator<<(double v) {
        char b[32];
        const int n = snprintf(b, sizeof b, "%g", v);
        s.append(b, (size_t)n);
        return *this;
    }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    SrcBuf &operator<<(T v) {
        char b[24];
        const auto r = std::to_chars(b, b + sizeof b, v);
        s.append(b, r.ptr);
        return *this;
    }
    std::string str() const { return s; }
};

std::string u64s(uint64_t x) {
    std::ostringstream o;
    o << x << "ull";
    return o.str();
}

std::string runs_expr(const char *src, int n, const uint8_t *s, const uint8_t *l, const uint8_t *d) {
    if (n == 0) return "0ull";
    std::ostringstream o;
    for (int i = 0; i < n; i++) {
        if (i) o << " | ";
        o << "((((u64)(" << src << ")) >> " << (int)s[i] << ") & " << u64s((l[i] >= 64) ? ~0ull : ((1ull << l[i]) - 1))
          << ") << " << (int)d[i];
    }
    return o.str();
}
}  // namespace

const JitConfig &jit_config() {
    static const JitConfig c = [] {
        JitConfig x;
        const char *e = getenv("HHLSV_JIT");
        if (!e) return x;
        std::string all(e);
        size_t pos = 0;
        while (pos <= all.size()) {
            size_t end = all.find(',', pos);
            if (end == std::string::npos) end = all.size();
            const std::string kv = all.substr(pos, end - pos);
            pos = end + 1;
            const size_t eq = kv.find('=');
            if (eq == std::string::npos) continue;
            const std::string key = kv.substr(0, eq), val = kv.substr(eq + 1);
            const int iv = atoi(val.c_str());
            if (key == "direct") x.direct = iv != 0;
            else if (key == "pf") x.prefetch = iv != 0;
            else if (key == "pfdist") x.pf_dist = std::max(1, iv);
            else if (key == "group") x.group = iv != 0;
            else if (key == "rtab") x.rtab = iv != 0;
            else if (key == "hoist") x.hoist = iv != 0;
            else if (key == "sparse") x.sparse = iv != 0;
            else if (key == "tail") x.tail = iv != 0;
            else if (key == "cw") x.cw = iv != 0;
            else if (key == "ctab") x.ctab = iv != 0;
            else if (key == "ctabbits") x.ctab_bits = std::max(0, std::min(6, iv));
            else if (key == "nbuf") x.nbuf = iv == 2 ? 2 : 1;
            else if (key == "minb") x.min_blocks = std::max(0, iv);
            else if (key == "mred") x.mred = iv != 0;
            else if (key == "spillfb") x.spillfb = iv != 0;
            else if (key == "dalap") x.dalap = std::max(0, iv);
            else if (key == "twiddle") x.twiddle = iv != 0;
            else if (key == "dmma") x.dmma = iv != 0;
            else if (key == "wrun") x.wrun = iv != 0;
            else if (key == "vdmma") x.vdmma = iv != 0;
            else if (key == "rb") x.reg_bits = (iv == 3) ? 3 : 4;
            else if (key == "skeleton") x.skeleton = iv != 0;
            else if (key == "xoverlap") x.xoverlap = iv != 0;
            else if (key == "graphs") x.graphs = iv != 0;
            else if (key == "ru") x.ru = std::max(0, iv);
            else if (key == "clobber") x.smem_clobber = iv != 0;
            else if (key == "ptxas") x.ptxas_opt = "-Xptxas=" + val;
            else if (key == "wmin") x.wmin = std::max(0, iv);
            else if (key == "dmerge") x.diag_merge = iv;
            else if (key == "echunk") x.eigen_chunk = std::max(0, iv);
            else if (key == "initfuse") x.init_fuse = iv != 0;
        }
        return x;
    }();
    return c;
}

bool jit_available(std::string *why) {
    Nvrtc &n = nvrtc();
    if (why) *why = n.why;
    return n.ok;
}

// ---------------------------------------------------------------- codegen ----
std::string gen_tile_kernel(const std::string &name, const dev::TileArgs &a, const std::vector<dev::RegPhase> &ph,
                            const std::vector<dev::RegOp> &ops, size_t *smem_extra, const InitSpec *init,
                            std::vector<std::pair<uint64_t, uint64_t>> *cwide, const std::vector<double2> *hblob,
                            const JitVariant &var) {
    const JitConfig &cfg = jit_config();
    const int T = a.T;
    const int RB = a.nreg, RA = 1 << RB;      // register bits / amplitudes per thread in a phase
    const int NTHR = 1 << (T - RB);
    const int SA = (T + 1) / 2, SB = T - SA;
    int wide_ops = 0;          // dense ops with >= 3 targets: unrolled when few, rolled (bounded code) when many
    for (auto &op : ops)
        if (op.kind == 0 && ((op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1)) >= 3)
            wide_ops++;
    // wide-op matrices staged once per (persistent) CTA in shared memory when few (<= 4 x 4 KB)
    // Wide-op matrices as constant-bank operands (DFMA reads them straight from the constant cache:
    // no shared-memory or L1 traffic for the matrix), up to 64 KB per pass module.
    std::map<int, size_t> cstage;      // op index -> offset (double2 units) in cw[]
    size_t ctot = 0;
    if (cwide && cfg.cw) {
        for (size_t i = 0; i < ops.size(); i++) {
            const auto &op = ops[i];
            const int Kk = (op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1);
            // as many as fit the kernel parameter space (32764 bytes); the rest read through L1
            if (op.kind == 0 && Kk >= 3 && ctot + ((size_t)1 << (2 * Kk)) <= 2040) {
                cstage[(int)i] = ctot;
                ctot += (size_t)1 << (2 * Kk);
            }
        }
        // small (1-, 2-qubit) dense matrices too, while space remains: their entries become constant-bank
        // DFMA operands instead of 2^2k preloaded registers (a pass of many 2-qubit ops -- Fig. 4 fused
        // transpiled streams -- otherwise spills kilobytes of registers)
        for (size_t i = 0; i < ops.size(); i++) {
            const auto &op = ops[i];
            const int Kk = (op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1);
            if (op.kind == 0 && Kk >= 1 && Kk <= 2 && ctot + ((size_t)1 << (2 * Kk)) <= 2040) {
                cstage[(int)i] = ctot;
                ctot += (size_t)1 << (2 * Kk);
            }
        }
        cwide->clear();
        std::vector<std::pair<size_t, int>> by_off;      // cw[] layout order = assigned offsets
        for (auto &kv : cstage) by_off.push_back({kv.second, kv.first});
        std::sort(by_off.begin(), by_off.end());
        for (auto &e : by_off) {
            const auto &op = ops[e.second];
            const int Kk = (op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1);
            cwide->push_back({op.data_off, (uint64_t)1 << (2 * Kk)});
        }
    }
    std::map<int, size_t> wstage;      // op index -> offset (double2 units) in the staging region
    size_t wtot = 0;
    if (wide_ops <= 4 && cstage.empty())
        for (size_t i = 0; i < ops.size(); i++) {
            const auto &op = ops[i];
            const int Kk = (op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1);
            if (op.kind == 0 && Kk >= 3) {
                wstage[(int)i] = wtot;
                wtot += (size_t)1 << (2 * Kk);
            }
        }
    // Runs of >= 2 consecutive diagonal ops inside a phase are precomposed per tile: the CTA
    // multiplies their tables, for the tile's fixed (out-of-tile) index bits, into a small
    // shared sub-table over the run's varying tile bits V; each amplitude then does ONE lookup
    // and ONE complex multiply for the whole run. Used when 2^|V| is small.
    struct DRun { int p, a, b; std::vector<int> V; size_t off; };
    std::vector<DRun> druns, rtabs;
    size_t dsub_max = 0;
    std::vector<size_t> used_ph;
    auto op_vary = [&](const dev::RegOp &op, const dev::RegPhase &P) {
        std::vector<int> v;
        for (int i = 0; i < RB; i++)
            if (op.ridx[1 << i]) v.push_back(P.R[i]);
        for (int r = 0; r < op.ntr; r++)
            for (int l = 0; l < op.t_len[r]; l++) v.push_back(op.t_src[r] + l);
        return v;
    };
    for (size_t p = 0; p < ph.size(); p++) {
        size_t used = 0;
        for (int oi = ph[p].op0; oi < ph[p].op1;) {
            if (ops[oi].kind != 1) {
                oi++;
                continue;
            }
            int oj = oi;
            std::vector<int> V;
            while (oj < ph[p].op1 && ops[oj].kind == 1) {
                for (int b : op_vary(ops[oj], ph[p]))
                    if (std::find(V.begin(), V.end(), b) == V.end()) V.push_back(b);
                oj++;
            }
            std::sort(V.begin(), V.end());
            if (oj - oi >= 2 && V.size() <= 9 && (int)V.size() <= T - 3) {
                druns.push_back({(int)p, oi, oj, V, used});
                used += (size_t)1 << V.size();
            }
            oi = oj;
        }
        // reciprocal rotation: its (s_m, c_m) pairs over the tile's clock bits precomputed per tile
        // (one division + square root per table entry instead of one per clock value per thread)
        for (int oi = ph[p].op0; oi < ph[p].op1; oi++) {
            if (ops[oi].kind != 2 || !cfg.rtab) continue;
            std::vector<int> V = op_vary(ops[oi], ph[p]);
            std::sort(V.begin(), V.end());
            if (V.size() <= 9 && (1u << V.size()) <= 2u * (1u << (T - RB))) {
                rtabs.push_back({(int)p, oi, oi + 1, V, used});
                used += (size_t)1 << V.size();
            }
        }
        dsub_max = std::max(dsub_max, used);
        used_ph.push_back(used);
    }
    // Small diagonal tables as constant-bank operands: a diagonal op (not in a precomposed run) whose
    // table index has no out-of-tile bits and at most 2 thread bits takes its entries from the by-value
    // kernel parameter (values per launch, like the wide matrices), chosen per thread by selects on its
    // thread bits: no L1/L2 table loads (their latency stalled the complex multiplies, ncu r02), no LSU
    // traffic. Only the entries the op's touched register slots can reach are passed.
    std::map<int, std::map<uint32_t, size_t>> ctab;     // op -> (table index -> position in cw[])
    auto tbits_of = [](const dev::RegOp &op) {           // (tile position, table bit) of the thread part
        std::vector<std::pair<int, int>> v;
        for (int r = 0; r < op.ntr; r++)
            for (int l = 0; l < op.t_len[r]; l++) v.push_back({op.t_src[r] + l, op.t_dst[r] + l});
        return v;
    };
    if (cwide && cfg.cw && cfg.ctab && !var.no_ctab) {
        for (size_t i = 0; i < ops.size(); i++) {
            const auto &op = ops[i];
            if (op.kind != 1 || op.ngr != 0) continue;
            bool in_run = false;
            for (auto &dr : druns) in_run |= (int)i >= dr.a && (int)i < dr.b;
            if (in_run) continue;
            const auto tbv = tbits_of(op);
            if ((int)tbv.size() > cfg.ctab_bits) continue;
            std::map<uint32_t, size_t> ent;
            for (int j = 0; j < RA; j++) {
                if ((j & op.rcm) != op.rcv) continue;
                for (uint32_t c = 0; c < (1u << tbv.size()); c++) {
                    uint32_t idx = op.ridx[j];
                    for (size_t b = 0; b < tbv.size(); b++)
                        if ((c >> b) & 1) idx |= 1u << tbv[b].second;
                    ent.emplace(idx, 0);
                }
            }
            if (ctot + ent.size() > 2040) continue;      // kernel parameter space: 32764 bytes
            for (auto &e : ent) {
                e.second = ctot++;
                cwide->push_back({op.data_off + e.first, 1});
            }
            ctab[(int)i] = std::move(ent);
        }
    }
    // table entry of diagonal op oi at register-slot index r; ibv = the op's runtime index variable
    auto dval = [&](int oi, uint32_t r, const std::string &ibv) -> std::string {
        const dev::RegOp &op = ops[oi];
        auto it = ctab.find(oi);
        if (it == ctab.end())
            return "__ldg(blob + " + std::to_string(op.data_off) + "ull + (" + ibv + " | " + std::to_string(r) + "u))";
        const auto tbv = tbits_of(op);
        std::function<std::string(size_t, uint32_t)> sel = [&](size_t b, uint32_t idx) -> std::string {
            if (b == tbv.size()) return "cwa.w[" + std::to_string(it->second.at(idx)) + "]";
            return "(((tb >> " + std::to_string(tbv[b].first) + ") & 1u) ? " + sel(b + 1, idx | (1u << tbv[b].second)) +
                   " : " + sel(b + 1, idx) + ")";
        };
        return sel(0, r);
    };
    // Hoisted sub-tables (default): phase p+1's tables are built at the end of phase p (the next
    // tile's phase-0 tables at the end of the last phase) into a region phase p-1 no longer reads,
    // so the barrier that ends phase p also publishes them: no separate barrier per sub-table build.
    // Regions alternate 0/1 by phase; with an odd phase count the last phase takes region 2.
    const size_t nph = ph.size();
    bool hoist = nph >= 2 && cfg.hoist;
    auto region = [&](size_t q) { return (nph % 2 == 1 && q + 1 == nph) ? 2 : (int)(q % 2); };
    if (hoist) {
        size_t R[3] = {0, 0, 0};
        for (size_t q = 0; q < nph; q++) R[region(q)] = std::max(R[region(q)], used_ph[q]);
        const size_t B[3] = {0, R[0], R[0] + R[1]};
        const size_t tot = R[0] + R[1] + R[2];
        // keep two CTAs per SM: (tile + dep tables + staging + sub-tables) <= 113 KB
        if (16 * ((size_t)1 << T) + 8 * (((size_t)1 << SA) + ((size_t)1 << SB)) + wtot * 16 + tot * 16 > 113 * 1024)
            hoist = false;
        else {
            for (auto &d : druns) d.off += B[region(d.p)];
            for (auto &d : rtabs) d.off += B[region(d.p)];
            dsub_max = tot;
        }
    }
    // Wide runs: >= 3 consecutive 4-qubit dense / controlled ops of a phase on exactly its 4 register bits
    // (e.g. the textbook QPE chain c-U^(2^j), all on the system register) whose conditions are only
    // out-of-tile (uniform per tile) and thread-bit controls over <= 2 thread bits. The CTA multiplies
    // the run's matrices per tile, for each assignment of those thread bits, into a 16 x 16 product
    // (one entry per thread per op: 16 complex FMAs, double-buffered tables in shared memory); each
    // thread then applies ONE matrix instead of up to N.
    struct WRun { int p, a, b; std::vector<int> V; };
    std::vector<WRun> wruns;
    if (cfg.wrun && RB == 4 && NTHR == 256 && !init)
        for (size_t p = 0; p < ph.size(); p++)
            for (int oi = ph[p].op0; oi < ph[p].op1;) {
                auto ok = [&](int q) {
                    const auto &op = ops[q];
                    return op.kind == 0 && op.mask == 15 && op.rcm == 0;
                };
                int oj = oi;
                std::vector<int> V;
                while (oj < ph[p].op1 && ok(oj)) {
                    for (int b = 0; b < 16; b++)
                        if (((ops[oj].tcm >> b) & 1) && std::find(V.begin(), V.end(), b) == V.end()) V.push_back(b);
                    if (V.size() > 2) break;
                    oj++;
                }
                if (oj - oi >= 3) {
                    std::vector<int> W;       // the thread bits of the ops actually in the run
                    for (int q = oi; q < oj; q++)
                        for (int b = 0; b < 16; b++)
                            if (((ops[q].tcm >> b) & 1) && std::find(W.begin(), W.end(), b) == W.end()) W.push_back(b);
                    wruns.push_back({(int)p, oi, oj, W});
                    oi = oj;
                } else {
                    oi = std::max(oi + 1, oj);
                }
            }
    size_t wtab_bytes = 0;            // 2 buffers x C combos x (256 + 1 pad) entries x 16 B
    for (auto &w : wruns) wtab_bytes = std::max(wtab_bytes, (size_t)2 * ((size_t)1 << w.V.size()) * 257 * 16);
    // Tile buffers: 1 = single buffer with several CTAs per SM overlapping each other's load and
    // compute phases (default; measured faster than double buffering at half the occupancy),
    // 2 = cp.async double buffering. Registers capped at 128/thread (16 warps per SM).
    int nbuf = (cfg.nbuf == 2 && !a.zload) ? 2 : 1;
    if (init) nbuf = 1;
    const size_t smem_cta = nbuf * 16 * ((size_t)1 << T) + 8 * (((size_t)1 << SA) + ((size_t)1 << SB)) + wtot * 16 +
                            dsub_max * 16 + wtab_bytes;
    if (smem_extra) *smem_extra = smem_cta;      // total dynamic shared memory of the kernel
    // resident CTAs per SM for __launch_bounds__: limited by shared memory, and by registers -- 128 per
    // thread for the 16 register amplitudes, allocated per WARP (a CTA smaller than a warp still takes
    // a whole warp): 65536 / (128 x 32) = 16 warps per SM. (Counting threads instead of warps gave a
    // 16-thread CTA a 64-register cap, an 11 KB spill stack and, at ptxas -O3, wrong amplitudes.)
    const int cta_warps = (NTHR + 31) / 32;
    const int reg_target = RB >= 4 ? 128 : 64;      // 16 or 8 register amplitudes per thread
    int min_blocks = std::max(1, std::min((int)((227 * 1024) / smem_cta), 65536 / (reg_target * 32 * cta_warps)));
    // Direct global I/O: when a phase's thread bits start with the tile's positions 0..2 and those are
    // the physical bits 0..2 (8 lanes cover 128 contiguous bytes), the first phase loads its 16
    // register amplitudes straight from HBM and the last phase stores them straight back; the tile
    // never passes through shared memory on the way in/out (saves 2 of the pass's smem sweeps
    // each way and the cp.async / store-loop address arithmetic).
    bool low3 = T >= 4 && a.tbits[0] == 0 && a.tbits[1] == 1 && a.tbits[2] == 2;
    low3 = low3 && cfg.direct;
    const bool din = nbuf == 1 && low3 && ph.front().R[0] >= 3;
    const bool pf_on = cfg.prefetch;
    auto sref = [&](int c) {       // shared-memory slot of register slot c (tile-local bits) in this phase
        std::ostringstream o;
        o << "cur[stb ^ " << swz_host((uint32_t)c) << "u]";
        return o.str();
    };
    const bool dout = nbuf == 1 && low3 && ph.back().R[0] >= 3;
    auto tb_expr = [&](const dev::RegPhase &P) {
        std::ostringstream o;
        o << "0u";
        for (int i = 0; i < T - RB; i++) o << " | (((threadIdx.x >> " << i << ") & 1u) << " << P.tpos[i] << ")";
        return o.str();
    };
    auto phys_slot = [&](const dev::RegPhase &P, int j) {      // physical offset of register slot j
        uint64_t c = 0;
        for (int i = 0; i < RB; i++)
            if ((j >> i) & 1) c |= 1ull << a.tbits[P.R[i]];
        return c;
    };
    if (cfg.min_blocks > 0) min_blocks = cfg.min_blocks;
    // Fused marginal (a.red >= 0): while the pass stores the final amplitudes each thread accumulates
    // Σ|a|² split by physical bit a.red (q0: bit 0, q1: bit 1) over all its tiles; at the end the CTA
    // combines its threads in a fixed order and writes red[2 blockIdx.x + {0, 1}] (summed by
    // k_pair_sum). Saves the readout's separate full-state read (16 B/amplitude).
    const bool red = a.red >= 0;
    const std::string rbs = std::to_string(a.red);
    SrcBuf k;
    if (ctot) k << "struct CWArg { double2 w[" << ctot << "]; };\n";
    k << "extern \"C\" __global__ void __launch_bounds__(" << NTHR << ", " << min_blocks << ") " << name
      << "(double2 *__restrict__ psi, const double2 *__restrict__ blob, u64 n_tiles, u64 rank_base, u64 tile0"
      << (red ? ", double *__restrict__ red" : "") << (ctot ? ", const CWArg cwa" : "") << ") {\n";
    k << "  constexpr u32 NT = " << (1u << T) << "u;\n";
    k << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n";
    k << "  const u32 sbase = (u32)__cvta_generic_to_shared(smem_raw);\n";
    k << "  const SArr buf0{sbase};\n  const SArr buf1{sbase + " << (nbuf == 2 ? "NT * 16u" : "0u") << "};\n";
    k << "  const SArr64 depA{sbase + " << nbuf << "u * NT * 16u};\n  const SArr64 depB{sbase + " << nbuf
      << "u * NT * 16u + " << (8 << SA) << "u};\n";
    k << "  for (int u = threadIdx.x; u < " << (1 << SA) << "; u += " << NTHR << ") { u64 d = 0;";
    for (int i = 0; i < SA; i++) k << " if (u & " << (1 << i) << ") d |= 1ull << " << a.tbits[i] << ";";
    k << " depA[u] = d; }\n";
    k << "  for (int u = threadIdx.x; u < " << (1 << SB) << "; u += " << NTHR << ") { u64 d = 0;";
    for (int i = 0; i < SB; i++) k << " if (u & " << (1 << i) << ") d |= 1ull << " << a.tbits[SA + i] << ";";
    k << " depB[u] = d; }\n";
    if (wtot) {
        k << "  const SArr wm{depB.b + " << (8 << SB) << "u};\n";
        for (auto &kv : wstage) {
            const auto &op = ops[kv.first];
            const int Kk = (op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1);
            if (op.is_signed)      // real matrix: column-major plain doubles
                k << "  for (int i = threadIdx.x; i < " << (1 << (2 * Kk)) << "; i += " << NTHR << ") stsd(wm.b + "
                  << kv.second * 16 << "u + (u32)(((i % " << (1 << Kk) << ") * " << (1 << Kk) << ") + i / " << (1 << Kk)
                  << ") * 8u, blob[" << op.data_off << "ull + i].x);\n";
            else
                k << "  for (int i = threadIdx.x; i < " << (1 << (2 * Kk)) << "; i += " << NTHR << ") wm[" << kv.second
                  << " + i] = blob[" << op.data_off << "ull + i];\n";
        }
    }
    if (dsub_max)
        k << "  const SArr dsub{depB.b + " << (8 << SB) << "u + " << wtot * 16 << "u};\n";
    if (wtab_bytes)
        k << "  const SArr wtab{depB.b + " << (8 << SB) << "u + " << (wtot * 16 + dsub_max * 16) << "u};\n";
    {   // tile index -> base: zeros inserted at the tile bits and at the skipped known-zero bits; lifted
        // bits (if any) take the top bits of the tile index
        std::vector<int> ins(a.tbits, a.tbits + T);
        for (int i = 0; i < a.nskip; i++) ins.push_back(a.skip[i]);
        for (int i = 0; i < a.nlift; i++) ins.push_back(a.lift[i]);
        std::sort(ins.begin(), ins.end());
        int ltiles = 0;
        while ((1ull << ltiles) < a.n_tiles) ltiles++;
        const int nlow = ltiles - a.nlift;
        k << "  auto tile_base = [](u64 t) { u64 b = " << (a.nlift ? "t & " + u64s((1ull << nlow) - 1ull) : std::string("t"))
          << ";";
        for (int b : ins) k << " b = insz(b, " << b << ");";
        for (int i = 0; i < a.nlift; i++) k << " b |= ((t >> " << nlow + i << ") & 1ull) << " << a.lift[i] << ";";
        k << " return b; };\n";
    }
    k << "  auto addr = [&](u64 base, u32 u) { return base | depA[u & " << ((1u << SA) - 1) << "u] | depB[u >> " << SA
      << "]; };\n";
    k << "  bar();\n";
    if (din) k << "  const u64 pd_in = addr(0ull, " << tb_expr(ph.front()) << ");\n";
    if (dout) k << "  const u64 pd_out = addr(0ull, " << tb_expr(ph.back()) << ");\n";
    auto emit_pre = [&](size_t pp, const std::string &gb) {     // per-tile sub-tables of phase pp
            const dev::RegPhase &Q = ph[pp];
            bool any_run = false;
            k << "      { const u64 gpre = " << gb << "; (void)gpre;\n";
        for (auto &dr : druns) {
            if (dr.p != (int)pp) continue;
            any_run = true;
            const int nv = (int)dr.V.size();
            k << "      for (u32 c = threadIdx.x; c < " << (1u << nv) << "u; c += " << NTHR << ") {\n        const u32 loc = 0u";
            for (int i = 0; i < nv; i++) k << " | (((c >> " << i << ") & 1u) << " << dr.V[i] << ")";
            k << ";\n        double2 acc = mk(1.0, 0.0);\n";
            for (int oi = dr.a; oi < dr.b; oi++) {
                const dev::RegOp &op = ops[oi];
                k << "        { const u64 ib = (" << runs_expr("gpre", op.ngr, op.g_src, op.g_len, op.g_dst) << ") | ("
                  << runs_expr("loc", op.ntr, op.t_src, op.t_len, op.t_dst) << ")";
                for (int i = 0; i < RB; i++)
                    if (op.ridx[1 << i]) {
                        int ob = 0;
                        while (!((op.ridx[1 << i] >> ob) & 1u)) ob++;
                        k << " | ((u64)((loc >> " << Q.R[i] << ") & 1u) << " << ob << ")";
                    }
                k << "; acc = cmul(acc, __ldg(blob + " << op.data_off << "ull + ib)); }\n";
            }
            k << "        dsub[" << dr.off << " + c] = acc;\n      }\n";
        }
        for (auto &rt : rtabs) {
            if (rt.p != (int)pp) continue;
            any_run = true;
            const dev::RegOp &op = ops[rt.a];
            const int nv = (int)rt.V.size();
            k << "      for (u32 c = threadIdx.x; c < " << (1u << nv) << "u; c += " << NTHR << ") {\n        const u32 loc = 0u";
            for (int i = 0; i < nv; i++) k << " | (((c >> " << i << ") & 1u) << " << rt.V[i] << ")";
            k << ";\n        const u64 m = (" << runs_expr("gpre", op.ngr, op.g_src, op.g_len, op.g_dst) << ") | ("
              << runs_expr("loc", op.ntr, op.t_src, op.t_len, op.t_dst) << ")";
            for (int i = 0; i < RB; i++)
                if (op.ridx[1 << i]) {
                    int ob = 0;
                    while (!((op.ridx[1 << i] >> ob) & 1u)) ob++;
                    k << " | ((u64)((loc >> " << Q.R[i] << ") & 1u) << " << ob << ")";
                }
            k << ";\n        const double2 pr = __ldg(blob + " << op.data_off << "ull);\n        const double s = recip_s(m, "
              << op.n_c << ", pr.x, " << op.is_signed << ", pr.y);\n        dsub[" << rt.off
              << " + c] = mk(s, sqrt(fma(-s, s, 1.0)));\n      }\n";
        }
            k << "      }\n";
            return any_run;
        };
    k << "  u64 tile = tile0 + blockIdx.x;      // tiles [tile0, n_tiles) of the pass\n";
    if (red) k << "  double q0 = 0.0, q1 = 0.0;      // fused marginal over bit " << a.red << "\n";
    if (hoist) {
        k << "  if (tile < n_tiles) {\n";
        emit_pre(0, "rank_base | tile_base(tile)");
        k << "  }\n  bar();\n";
    }
    if (nbuf == 2) {
        k << "  if (tile < n_tiles) { const u64 b0 = tile_base(tile); for (u32 u = threadIdx.x; u < NT; u += " << NTHR
          << ") cp_async16s(buf0.at(swz(u)), &psi[addr(b0, u)]); }\n";
        k << "  cp_async_commit();\n";
        k << "  for (int it = 0; tile < n_tiles; tile += gridDim.x, it++) {\n";
        k << "    const SArr cur = (it & 1) ? buf1 : buf0;\n    const SArr nxt = (it & 1) ? buf0 : buf1;\n";
        k << "    const u64 next = tile + gridDim.x;\n";
        k << "    if (next < n_tiles) { const u64 b1 = tile_base(next); for (u32 u = threadIdx.x; u < NT; u += " << NTHR
          << ") cp_async16s(nxt.at(swz(u)), &psi[addr(b1, u)]); }\n";
        k << "    cp_async_commit();\n";
        k << "    const u64 base = tile_base(tile);\n    const u64 gbase = rank_base | base;\n    (void)gbase;\n";
        k << "    cp_async_wait1();\n    bar();\n";
    } else {
        k << "  for (; tile < n_tiles; tile += gridDim.x) {\n";
        k << "    const SArr cur = buf0;\n";
        k << "    const u64 base = tile_base(tile);\n    const u64 gbase = rank_base | base;\n    (void)gbase;\n";
        // L2 prefetch of this CTA's next tile: its HBM reads overlap this tile's compute, and the
        // next tile's loads then hit L2 (296 CTAs x 64 KB in flight << 126 MB L2)
        if (pf_on && !init) {
            const int pfd = std::max(1, cfg.pf_dist);
            k << "    if (tile + " << pfd << "ull * gridDim.x < n_tiles) {\n      const u64 nb = tile_base(tile + " << pfd
              << "ull * gridDim.x);\n";
            if (din) {       // known-zero slots (zload) are never read: not prefetched either
                uint32_t rz0 = 0;
                for (int i = 0; i < RB; i++) rz0 |= 1u << ph.front().R[i];
                const bool thr_z = (a.zload & ~rz0) != 0;
                k << "      if ((threadIdx.x & 7u) == 0u" << (thr_z ? " && !((" + tb_expr(ph.front()) + ") & " +
                                                                       std::to_string(a.zload) + "u)" : std::string())
                  << ") { const char *g = (const char *)(psi + (nb | pd_in));";
                for (int j = 0; j < RA; j++) {
                    uint32_t rdj = 0;
                    for (int i = 0; i < RB; i++)
                        if ((j >> i) & 1) rdj |= 1u << ph.front().R[i];
                    if (rdj & a.zload) continue;
                    k << " pf_l2(g + " << u64s(16 * phys_slot(ph.front(), j)) << ");";
                }
                k << " }\n";
            } else {
                k << "      for (u32 u = threadIdx.x * 8u; u < NT; u += " << 8 * NTHR << "u) "
                  << (a.zload ? "if (!(u & " + std::to_string(a.zload) + "u)) " : std::string())
                  << "pf_l2(psi + addr(nb, u));\n";
            }
            k << "    }\n";
        }
        if (din) {
            // phase 0 reads (or, fused init, computes) its registers directly
        } else if (init) {      // fused product-state init: compute the tile instead of reading it
            k << "    for (u32 u = threadIdx.x; u < NT; u += " << NTHR << ") {\n      const u64 gi = gbase | addr(0ull, u);\n";
            k << "      double2 amp = mk(0.0, 0.0);\n      if (!(gi & " << u64s(init->zero_mask) << ")) {\n";
            for (size_t g = 0; g < init->off.size(); g++) {
                // runs of consecutive bits: table bit j <- physical bit bits[j]
                const auto &B = init->bits[g];
                std::vector<uint8_t> src, len, dst;
                for (size_t j = 0; j < B.size(); j++) {
                    if (!src.empty() && B[j] == src.back() + len.back()) {
                        len.back()++;
                        continue;
                    }
                    src.push_back((uint8_t)B[j]);
                    dst.push_back((uint8_t)j);
                    len.push_back(1);
                }
                k << "        const double2 t" << g << " = __ldg(blob + " << init->off[g] << "ull + ("
                  << runs_expr("gi", (int)src.size(), src.data(), len.data(), dst.data()) << "));\n";
                k << "        amp = " << (g == 0 ? std::string("t0") : "cmul(amp, t" + std::to_string(g) + ")") << ";\n";
            }
            k << "      }\n      cur[swz(u)] = amp;\n    }\n    bar();\n";
        } else {
            if (a.zload)      // known-zero slots are not read
                k << "    for (u32 u = threadIdx.x; u < NT; u += " << NTHR << ") { if (u & " << a.zload
                  << "u) cur[swz(u)] = mk(0.0, 0.0); else cp_async16s(cur.at(swz(u)), &psi[addr(base, u)]); }\n";
            else
                k << "    for (u32 u = threadIdx.x; u < NT; u += " << NTHR << ") cp_async16s(cur.at(swz(u)), &psi[addr(base, u)]);\n";
            k << "    cp_async_commit();\n    cp_async_wait0();\n    bar();\n";
        }
    }
    for (size_t p = 0; p < ph.size(); p++) {
        const dev::RegPhase &P = ph[p];
        k << "    { // phase " << p << "\n      const u32 tb = 0u";
        for (int i = 0; i < T - RB; i++) k << " | (((threadIdx.x >> " << i << ") & 1u) << " << P.tpos[i] << ")";
        k << ";\n";
        // the swizzle is XOR-linear and tb / slot bits are disjoint: swz(tb | c) = swz(tb) ^ swz(c), so a
        // register slot's shared-memory index is one XOR with a codegen constant
        k << "      const u32 stb = swz(tb);\n";
        int rd[16];
        for (int j = 0; j < RA; j++) {
            rd[j] = 0;
            for (int i = 0; i < RB; i++)
                if ((j >> i) & 1) rd[j] |= 1 << P.R[i];
        }
        if (!hoist) {
            if (emit_pre(p, "gbase")) k << "      bar();\n";
        }

        // Tail on the FP64 tensor cores: the last phase (stored through shared memory) holds ONE real,
        // unconditioned 4-qubit dense op on exactly its register bits (the final V of the HHL program).
        // Per warp it is Y = V X with X = the 32 groups' 16 amplitudes as 64 real columns (re, im):
        // 2 row tiles x 4 k-steps x 8 column tiles of mma.m8n8k4.f64, operands straight from the tile in
        // shared memory (lane (n, kk) reads amplitude kk + 4 ks of group (8 ct + n) / 2), results written
        // back in place (a column tile's groups are read only by its own mma) for the final store loop.
        bool vdm = false;
        if (cfg.vdmma && p + 1 == ph.size() && !dout && P.op1 - P.op0 == 1 && NTHR == 256 && RB == 4) {
            const dev::RegOp &op = ops[P.op0];
            vdm = op.kind == 0 && op.mask == 15 && op.is_signed && !op.rcm && !op.tcm && !op.gcm;
        }
        if (vdm) {
            const dev::RegOp &op = ops[P.op0];
            auto cs = cstage.find(P.op0);
            auto ventry = [&](const std::string &idx) {
                if (cs != cstage.end()) return "cwa.w[" + std::to_string(cs->second) + "u + " + idx + "].x";
                return "__ldg(&blob[" + std::to_string(op.data_off) + "ull + " + idx + "].x)";
            };
            k << "      { // op " << P.op0 << " on the FP64 tensor cores (DMMA)\n";
            k << "        auto tbf = [](u32 t) { return 0u";
            for (int i = 0; i < T - RB; i++) k << " | (((t >> " << i << ") & 1u) << " << P.tpos[i] << ")";
            k << "; };\n";
            k << "        const u32 lane = threadIdx.x & 31u, wbase = threadIdx.x & ~31u, n = lane >> 2, kk = lane & 3u;\n";
            k << "        double a[2][4];\n";
            for (int rt = 0; rt < 2; rt++)
                for (int ks = 0; ks < 4; ks++)
                    k << "        a[" << rt << "][" << ks << "] = " << ventry("(" + std::to_string(8 * rt) + "u + n) * 16u + " + std::to_string(4 * ks) + "u + kk") << ";\n";
            k << "        auto rdf = [](u32 j) { return 0u";        // register slot j -> tile-local offset
            for (int i = 0; i < 4; i++) k << " | (((j >> " << i << ") & 1u) << " << P.R[i] << ")";
            k << "; };\n";
            // two column tiles per iteration: 4 independent accumulator chains; B fragments as single
            // 8-byte shared loads (re or im of one amplitude)
            k << "        #pragma unroll 1\n        for (u32 ct = 0; ct < 8u; ct += 2u) {\n";
            k << "          double b[2][4], d[2][2][2];\n";
            k << "          #pragma unroll\n          for (int c2 = 0; c2 < 2; c2++) {\n";
            k << "            const u32 gi = tbf(wbase + 4u * (ct + c2) + (n >> 1));   // B column: group, part\n";
            k << "            #pragma unroll\n            for (int ks = 0; ks < 4; ks++) b[c2][ks] = ldsd(cur.b + (swz(gi | rdf(4u * ks + kk)) << 4) + ((n & 1u) << 3));\n";
            k << "            d[c2][0][0] = d[c2][0][1] = d[c2][1][0] = d[c2][1][1] = 0.0;\n          }\n";
            k << "          #pragma unroll\n          for (int ks = 0; ks < 4; ks++)\n";
            k << "            #pragma unroll\n            for (int c2 = 0; c2 < 2; c2++)\n";
            k << "              #pragma unroll\n              for (int rt = 0; rt < 2; rt++) dmma884(d[c2][rt][0], d[c2][rt][1], a[rt][ks], b[c2][ks]);\n";
            k << "          #pragma unroll\n          for (int c2 = 0; c2 < 2; c2++) {\n";
            k << "            const u32 go = tbf(wbase + 4u * (ct + c2) + kk);      // D columns: group (re, im)\n";
            k << "            #pragma unroll\n            for (int rt = 0; rt < 2; rt++) cur[swz(go | rdf(8u * rt + n))] = mk(d[c2][rt][0], d[c2][rt][1]);\n";
            k << "          }\n        }\n      }\n";
        } else if (p == 0 && din && init) {
            for (int j = 0; j < RA; j++) {
                k << "      double2 v" << j << " = mk(0.0, 0.0);\n      { const u64 gi = gbase | pd_in | " << u64s(phys_slot(P, j))
                  << ";\n        if (!(gi & " << u64s(init->zero_mask) << ")) {\n";
                for (size_t g = 0; g < init->off.size(); g++) {
                    const auto &B = init->bits[g];
                    std::vector<uint8_t> src, len, dst;
                    for (size_t q = 0; q < B.size(); q++) {
                        if (!src.empty() && B[q] == src.back() + len.back()) {
                            len.back()++;
                            continue;
                        }
                        src.push_back((uint8_t)B[q]);
                        dst.push_back((uint8_t)q);
                        len.push_back(1);
                    }
                    k << "          const double2 t" << g << " = __ldg(blob + " << init->off[g] << "ull + ("
                      << runs_expr("gi", (int)src.size(), src.data(), len.data(), dst.data()) << "));\n";
                    k << "          v" << j << " = " << (g == 0 ? std::string("t0") : "cmul(v" + std::to_string(j) + ", t" + std::to_string(g) + ")")
                      << ";\n";
                }
                k << "        }\n      }\n";
            }
        } else if (p == 0 && din) {
            k << "      const double2 *gin = psi + (base | pd_in);\n";
            for (int j = 0; j < RA; j++) {
                // known-zero slots (zload) are not read: register part decided at codegen, thread part per thread
                if ((uint32_t)rd[j] & a.zload) k << "      double2 v" << j << " = mk(0.0, 0.0);\n";
                else if (a.zload)
                    k << "      double2 v" << j << " = (tb & " << a.zload << "u) ? mk(0.0, 0.0) : ldcs_v(gin + "
                      << u64s(phys_slot(P, j)) << ");\n";
                else k << "      double2 v" << j << " = ldcs_v(gin + " << u64s(phys_slot(P, j)) << ");\n";
            }
        } else {
            for (int j = 0; j < RA; j++) k << "      double2 v" << j << " = " << sref(rd[j]) << ";\n";
        }
        // The last op of a last phase that stores through shared memory is a wide dense op without
        // controls: its rows are written to their final shared-memory slots, so neither the register
        // reload nor the end-of-phase stores are needed.
        bool tail_in_smem = vdm;      // the DMMA tail wrote its results to their smem slots
        auto tail_wide = [&](int oi) {
            const dev::RegOp &op = ops[oi];
            const int Kq = (op.mask & 1) + ((op.mask >> 1) & 1) + ((op.mask >> 2) & 1) + ((op.mask >> 3) & 1);
            return p + 1 == ph.size() && !dout && oi + 1 == P.op1 && op.kind == 0 && Kq >= 3 && !op.rcm && !op.tcm &&
                   !op.gcm && cfg.tail;
        };
        // Twiddle-butterfly fusion: the last complex multiply a diagonal group / op applies to the
        // x1 slot of the butterfly that follows it (Hadamard on the bit the phases are conditioned on,
        // as in every (I)QFT stage: CP ladder / eigen-phase, then H) is kept pending and folded into
        // that butterfly: (x0 + w x1, 2 x0 - (x0 + w x1)) costs 6 FP64 ops per pair instead of 8.
        std::map<int, std::string> pend;          // slot -> pending factor variable
        auto flush = [&](int j) {
            auto it = pend.find(j);
            if (it == pend.end()) return;
            k << "      v" << j << " = cmul(" << it->second << ", v" << j << ");\n";
            pend.erase(it);
        };
        auto flush_all = [&] {
            while (!pend.empty()) flush(pend.begin()->first);
        };
        int npend = 0;
        // butterfly bit of op q if it can absorb pending x1 factors (unconditional kind-4 op), else -1
        auto bfly_bit = [&](int q) {
            if (!cfg.twiddle || q >= P.op1 || ops[q].kind != 4 || ops[q].gcm || ops[q].tcm) return -1;
            int A = 0;
            while (!((ops[q].mask >> A) & 1)) A++;
            return A;
        };
        auto emit_single = [&](int oi) {
            tail_in_smem = tail_wide(oi);
            const dev::RegOp &op = ops[oi];
            if (op.kind != 4) flush_all();
            else {
                int A = 0;
                while (!((op.mask >> A) & 1)) A++;
                std::vector<int> keep;
                for (auto &kv : pend)
                    if (!((kv.first >> A) & 1) || op.gcm || op.tcm) keep.push_back(kv.first);
                for (int j : keep) flush(j);
            }
            std::ostringstream cond;
            if (op.gcm) cond << "((gbase & " << u64s(op.gcm) << ") == " << u64s(op.gcv) << ")";
            if ((op.kind == 0 || op.kind == 1) && op.tcm) {
                if (op.gcm) cond << " && ";
                cond << "((tb & " << op.tcm << "u) == " << op.tcv << "u)";
            }
            const std::string c = cond.str();
            // pending factors of a diagonal op folded into the next butterfly (declared outside the block)
            const int Ab = (op.kind == 1 && c.empty()) ? bfly_bit(oi + 1) : -1;
            const int pid = npend;
            if (Ab >= 0) {
                npend++;
                for (int j = 0; j < RA; j++)
                    if ((j & op.rcm) == op.rcv && ((j >> Ab) & 1)) k << "      double2 pw" << pid << "_" << j << ";\n";
            }
            k << "      " << (c.empty() ? "{" : "if (" + c + ") {") << " // op " << oi << "\n";
            if (op.kind == 3) {          // deferred global scale
                k << "        const double sc = __ldg(&blob[" << op.data_off << "ull].x);\n";
                for (int j = 0; j < RA; j++) k << "        v" << j << " = mk(v" << j << ".x * sc, v" << j << ".y * sc);\n";
            } else if (op.kind == 4) {   // unscaled butterfly (Hadamard-like gate)
                int A = 0;
                while (!((op.mask >> A) & 1)) A++;
                for (int j = 0; j < RA; j++) {
                    if ((j >> A) & 1) continue;
                    const int j1 = j | (1 << A);
                    auto pw = pend.find(j1);
                    if (pw != pend.end()) {      // fused: s = x0 + w x1, x1' = 2 x0 - s
                        const std::string &w = pw->second;
                        k << "        { const double2 x0 = v" << j << ", x1 = v" << j1 << "; const double2 s = mk(fma("
                          << w << ".x, x1.x, fma(-" << w << ".y, x1.y, x0.x)), fma(" << w << ".x, x1.y, fma(" << w
                          << ".y, x1.x, x0.y))); v" << j1 << " = mk(fma(2.0, x0.x, -s.x), fma(2.0, x0.y, -s.y)); v" << j
                          << " = s; }\n";
                        pend.erase(pw);
                        continue;
                    }
                    k << "        { const double2 x0 = v" << j << ", x1 = v" << j1 << "; v" << j
                      << " = mk(x0.x + x1.x, x0.y + x1.y); v" << j1 << " = mk(x0.x - x1.x, x0.y - x1.y); }\n";
                }
            } else if (op.kind == 0) {
                const int M = op.mask;
                int K = 0;
                for (int i = 0; i < 4; i++) K += (M >> i) & 1;
                const int D = 1 << K;
                const bool real = op.is_signed != 0;
                k << "        const double2 *U = blob + " << op.data_off << "ull;\n";
                const auto csK = cstage.find(oi);          // small matrix in the constant bank?
                if (K <= 2 && csK == cstage.end())
                    for (int i = 0; i < D * D; i++) k << "        const double2 u" << i << " = __ldg(U + " << i << ");\n";
                for (int g = 0; g < RA; g++) {
                    if (g & M) continue;
                    if ((g & op.rcm) != op.rcv) continue;
                    if (K >= 3) {
                        // wide op: inputs straight from the v registers, each output row goes to this
                        // thread's own smem slot, then the D slots are reloaded (no input copies: keeps
                        // the pass's register footprint, hence occupancy, unchanged)
                        int Rpos[4], nrp = 0;
                        for (int i = 0; i < 4; i++)
                            if ((M >> i) & 1) Rpos[nrp++] = P.R[i];
                        auto row = [&](const std::string &Ur) {
                            std::ostringstream o;
                            for (int cc = 0; cc < D; cc++) {
                                const std::string in = "v" + std::to_string(g | dep_slot(cc, M));
                                if (real)
                                    o << " { const double w = __ldg(&" << Ur << "[" << cc << "].x); ax = fma(w, " << in
                                      << ".x, ax); ay = fma(w, " << in << ".y, ay); }";
                                else
                                    o << " { const double2 w = __ldg(" << Ur << " + " << cc << "); ax = fma(w.x, " << in
                                      << ".x, ax); ax = fma(-w.y, " << in << ".y, ax); ay = fma(w.x, " << in
                                      << ".y, ay); ay = fma(w.y, " << in << ".x, ay); }";
                            }
                            return o.str();
                        };
                        auto row_s = [&](const std::string &Ur) {      // matrix row in shared memory
                            std::ostringstream o;
                            for (int cc = 0; cc < D; cc++) {
                                const std::string in = "v" + std::to_string(g | dep_slot(cc, M));
                                if (real)
                                    o << " { const double w = ((double2)" << Ur << "[" << cc << "]).x; ax = fma(w, " << in
                                      << ".x, ax); ay = fma(w, " << in << ".y, ay); }";
                                else
                                    o << " { const double2 w = " << Ur << "[" << cc << "]; ax = fma(w.x, " << in
                                      << ".x, ax); ax = fma(-w.y, " << in << ".y, ax); ay = fma(w.x, " << in
                                      << ".y, ay); ay = fma(w.y, " << in << ".x, ay); }";
                            }
                            return o.str();
                        };
                        k << "        {\n";
                        auto ws0 = wstage.find(oi);
                        auto cs0 = cstage.find(oi);
                        if (cs0 != cstage.end()) {
                            // rolled loop over blocks of RU rows; matrix entries from the by-value kernel
                            // parameter (constant bank, uniform across the warp)
                            const int RU = std::min(D, cfg.ru > 0 ? cfg.ru : (real ? 16 : 2));   // measured: real 16 best
                            k << "          #pragma unroll 1\n          for (int r = 0; r < " << D << "; r += " << RU << ") {";
                            for (int q = 0; q < RU; q++) k << " double ax" << q << " = 0.0, ay" << q << " = 0.0;";
                            k << "\n";
                            for (int cc = 0; cc < D; cc++) {
                                const std::string in = "v" + std::to_string(g | dep_slot(cc, M));
                                for (int q = 0; q < RU; q++) {
                                    // one row block (RU == D): exact structural zeros of the matrix (e.g. the
                                    // identity padding of the system register in V) are skipped at codegen
                                    if (hblob && RU == D && cfg.sparse) {
                                        const double2 e = (*hblob)[op.data_off + (size_t)q * D + cc];
                                        if (e.x == 0.0 && e.y == 0.0) continue;
                                    }
                                    const std::string w = "cwa.w[" + std::to_string(cs0->second + cc) + " + (r + " + std::to_string(q) +
                                                          ") * " + std::to_string(D) + "]";
                                    if (real)
                                        k << "            { const double w = " << w << ".x; ax" << q << " = fma(w, " << in << ".x, ax" << q
                                          << "); ay" << q << " = fma(w, " << in << ".y, ay" << q << "); }\n";
                                    else
                                        k << "            { const double2 w = " << w << "; ax" << q << " = fma(w.x, " << in << ".x, ax" << q
                                          << "); ax" << q << " = fma(-w.y, " << in << ".y, ax" << q << "); ay" << q << " = fma(w.x, " << in
                                          << ".y, ay" << q << "); ay" << q << " = fma(w.y, " << in << ".x, ay" << q << "); }\n";
                                }
                            }
                            for (int q = 0; q < RU; q++) {
                                k << "            { const u32 rr = (u32)r + " << q << "u; const u32 slot = " << rd[g] << "u";
                                for (int i = 0; i < K; i++) k << " | ((rr >> " << i << ") & 1u) << " << Rpos[i];
                                k << "; cur[swz(tb | slot)] = mk(ax" << q << ", ay" << q << "); }\n";
                            }
                            k << "          }\n";
                        } else if (ws0 != wstage.end()) {
                            // rolled loop over blocks of RU rows with RU independent accumulator pairs
                            // (ILP for the FMA chains); a real matrix is staged column-major as plain
                            // doubles so one 16-byte shared load feeds two rows
                            const int RU = real ? 4 : 2;
                            const std::string wb = "wm.b + " + std::to_string(ws0->second * 16) + "u";
                            k << "          #pragma unroll 1\n          for (int r = 0; r < " << D << "; r += " << RU << ") {";
                            for (int q = 0; q < RU; q++) k << " double ax" << q << " = 0.0, ay" << q << " = 0.0;";
                            k << "\n";
                            for (int cc = 0; cc < D; cc++) {
                                const std::string in = "v" + std::to_string(g | dep_slot(cc, M));
                                if (real) {
                                    k << "            { const u32 wa = " << wb << " + (u32)(" << cc * D << " + r) * 8u; const double2 w01 = lds(wa), w23 = lds(wa + 16u);"
                                      << " ax0 = fma(w01.x, " << in << ".x, ax0); ay0 = fma(w01.x, " << in << ".y, ay0);"
                                      << " ax1 = fma(w01.y, " << in << ".x, ax1); ay1 = fma(w01.y, " << in << ".y, ay1);"
                                      << " ax2 = fma(w23.x, " << in << ".x, ax2); ay2 = fma(w23.x, " << in << ".y, ay2);"
                                      << " ax3 = fma(w23.y, " << in << ".x, ax3); ay3 = fma(w23.y, " << in << ".y, ay3); }\n";
                                } else {
                                    for (int q = 0; q < RU; q++)
                                        k << "            { const double2 w = lds(" << wb << " + (u32)((r + " << q << ") * " << D << " + " << cc
                                          << ") * 16u); ax" << q << " = fma(w.x, " << in << ".x, ax" << q << "); ax" << q << " = fma(-w.y, "
                                          << in << ".y, ax" << q << "); ay" << q << " = fma(w.x, " << in << ".y, ay" << q << "); ay" << q
                                          << " = fma(w.y, " << in << ".x, ay" << q << "); }\n";
                                }
                            }
                            for (int q = 0; q < RU; q++) {
                                k << "            { const u32 rr = (u32)r + " << q << "u; const u32 slot = " << rd[g] << "u";
                                for (int i = 0; i < K; i++) k << " | ((rr >> " << i << ") & 1u) << " << Rpos[i];
                                k << "; cur[swz(tb | slot)] = mk(ax" << q << ", ay" << q << "); }\n";
                            }
                            k << "          }\n";
                        } else {   // rolled row loop: bounded registers (inputs stay in v) and code size
                            k << "          #pragma unroll 1\n          for (int r = 0; r < " << D
                              << "; r++) { double ax = 0.0, ay = 0.0; const auto Ur = "
                              << (ws0 != wstage.end() ? "wm + " + std::to_string(ws0->second) + "u" : std::string("U"))
                              << " + r * " << D << ";" << (ws0 != wstage.end() ? row_s("Ur") : row("Ur"))
                              << " const u32 slot = " << rd[g] << "u";
                            for (int i = 0; i < K; i++) k << " | (((u32)r >> " << i << ") & 1u) << " << Rpos[i];
                            k << "; cur[swz(tb | slot)] = mk(ax, ay); }\n";
                        }
                        if (!tail_in_smem)      // else: the outputs already sit in their final smem slots
                            for (int r = 0; r < D; r++) {
                                const int j = g | dep_slot(r, M);
                                k << "          v" << j << " = " << sref(rd[j]) << ";\n";
                            }
                        k << "        }\n";
                        continue;
                    }
                    k << "        {";
                    for (int cc = 0; cc < D; cc++) k << " const double2 i" << cc << " = v" << (g | dep_slot(cc, M)) << ";";
                    k << "\n";
                    for (int r = 0; r < D; r++) {
                        k << "          { double ax = 0.0, ay = 0.0;";
                        for (int cc = 0; cc < D; cc++) {
                            std::string u = (K <= 2 && csK != cstage.end())
                                                ? ("cwa.w[" + std::to_string(csK->second + (size_t)r * D + cc) + "]")
                                            : K <= 2 ? ("u" + std::to_string(r * D + cc))
                                                     : ("__ldg(U + " + std::to_string(r * D + cc) + ")");
                            if (real) {
                                k << " ax = fma(" << u << ".x, i" << cc << ".x, ax); ay = fma(" << u << ".x, i" << cc
                                  << ".y, ay);";
                            } else {
                                k << " { const double2 w = " << u << "; ax = fma(w.x, i" << cc << ".x, ax); ax = fma(-w.y, i"
                                  << cc << ".y, ax); ay = fma(w.x, i" << cc << ".y, ay); ay = fma(w.y, i" << cc
                                  << ".x, ay); }";
                            }
                        }
                        k << " v" << (g | dep_slot(r, M)) << " = mk(ax, ay); }\n";
                    }
                    k << "        }\n";
                }
            } else {
                k << "        const u64 ib = (" << runs_expr("gbase", op.ngr, op.g_src, op.g_len, op.g_dst) << ") | ("
                  << runs_expr("tb", op.ntr, op.t_src, op.t_len, op.t_dst) << ");\n";
                if (op.kind == 1) {
                    const int A = Ab;
                    for (int j = 0; j < RA; j++)
                        if ((j & op.rcm) == op.rcv)
                            k << "        const double2 d" << j << " = " << dval(oi, op.ridx[j], "ib") << ";\n";
                    for (int j = 0; j < RA; j++) {
                        if ((j & op.rcm) != op.rcv) continue;
                        if (A >= 0 && ((j >> A) & 1)) {
                            const std::string w = "pw" + std::to_string(pid) + "_" + std::to_string(j);
                            k << "        " << w << " = d" << j << ";\n";
                            pend[j] = w;
                        } else {
                            k << "        v" << j << " = cmul(d" << j << ", v" << j << ");\n";
                        }
                    }
                } else {
                    int A = 0;
                    while (!((op.mask >> A) & 1)) A++;
                    const DRun *rt = nullptr;
                    for (auto &r : rtabs)
                        if (r.a == oi) rt = &r;
                    if (!rt) k << "        const double2 pr = __ldg(blob + " << op.data_off << "ull);\n";
                    else {
                        k << "        const u32 bt = 0u";
                        for (size_t i = 0; i < rt->V.size(); i++)
                            if (std::find(P.R, P.R + RB, rt->V[i]) == P.R + RB)
                                k << " | (((tb >> " << rt->V[i] << ") & 1u) << " << i << ")";
                        k << ";\n";
                    }
                    // one division + square root per distinct clock value among the slot pairs
                    // (once per thread when no clock bit is a register bit), or one lookup in the
                    // tile's precomputed (s, c) table
                    std::map<uint32_t, int> sc;
                    for (int j = 0; j < RA; j++) {
                        if ((j >> A) & 1) continue;
                        if (sc.count(op.ridx[j])) continue;
                        const int id = (int)sc.size();
                        sc[op.ridx[j]] = id;
                        if (rt) {
                            int cj = 0;
                            for (size_t i = 0; i < rt->V.size(); i++)
                                for (int r = 0; r < RB; r++)
                                    if (P.R[r] == rt->V[i] && ((j >> r) & 1)) cj |= 1 << i;
                            k << "        const double2 sc" << id << " = dsub[" << rt->off << " + (bt | " << cj
                              << "u)]; const double s" << id << " = sc" << id << ".x, c" << id << " = sc" << id << ".y;\n";
                        } else {
                            k << "        const double s" << id << " = recip_s(ib | " << op.ridx[j] << "u, " << op.n_c
                              << ", pr.x, " << op.is_signed << ", pr.y); const double c" << id << " = sqrt(fma(-s" << id
                              << ", s" << id << ", 1.0));\n";
                        }
                    }
                    for (int j = 0; j < RA; j++) {
                        if ((j >> A) & 1) continue;
                        const int j1 = j | (1 << A);
                        const std::string s = "s" + std::to_string(sc[op.ridx[j]]);
                        const std::string c = "c" + std::to_string(sc[op.ridx[j]]);
                        k << "        { const double2 x0 = v" << j << ", x1 = v" << j1 << "; v" << j << " = mk(" << c
                          << " * x0.x - " << s << " * x1.x, " << c << " * x0.y - " << s << " * x1.y); v" << j1
                          << " = mk(" << s << " * x0.x + " << c << " * x1.x, " << s << " * x0.y + " << c
                          << " * x1.y); }\n";
                    }
                }
            }
            k << "      }\n";
        };
        // Consecutive diagonal ops (not precomposed in a run) whose only conditions are register-slot
        // controls are applied as ONE group: ops whose table value is the same on every slot they
        // touch (e.g. CP-ladder chunks over thread / out-of-tile bits) are multiplied into one scalar
        // per distinct slot set, and each slot then takes one complex multiply per distinct factor
        // list (shared across slots) instead of one per op.
        auto op_cond = [&](const dev::RegOp &op) {     // thread / tile guard of a diagonal op ("" = none)
            std::ostringstream c;
            if (op.gcm) c << "((gbase & " << u64s(op.gcm) << ") == " << u64s(op.gcv) << ")";
            if (op.tcm) {
                if (op.gcm) c << " && ";
                c << "((tb & " << op.tcm << "u) == " << op.tcv << "u)";
            }
            return c.str();
        };
        auto emit_group = [&](const std::vector<int> &G, int A) {
            flush_all();
            const int pid = npend;
            if (A >= 0) {        // pending factors of the x1 slots (declared outside the block)
                npend++;
                for (int j = 0; j < RA; j++)
                    if ((j >> A) & 1) k << "      double2 pw" << pid << "_" << j << ";\n";
            }
            k << "      { // diagonal group of " << G.size() << " ops\n";
            std::vector<std::vector<std::string>> fac(16);
            std::map<uint32_t, std::vector<int>> uni;
            std::vector<int> var;
            for (int oi : G) {
                const dev::RegOp &op = ops[oi];
                k << "        const u64 ib" << oi << " = (" << runs_expr("gbase", op.ngr, op.g_src, op.g_len, op.g_dst)
                  << ") | (" << runs_expr("tb", op.ntr, op.t_src, op.t_len, op.t_dst) << ");\n";
                uint32_t m = 0;
                std::vector<uint32_t> rs;
                for (int j = 0; j < RA; j++)
                    if ((j & op.rcm) == op.rcv) {
                        m |= 1u << j;
                        if (std::find(rs.begin(), rs.end(), op.ridx[j]) == rs.end()) rs.push_back(op.ridx[j]);
                    }
                if (rs.size() == 1) uni[m].push_back(oi);
                else var.push_back(oi);
            }
            int nu = 0;
            for (auto &kv : uni) {
                const std::string U = "U" + std::to_string(nu++);
                bool first = true;
                for (int oi : kv.second) {
                    const dev::RegOp &op = ops[oi];
                    int j0 = 0;
                    while (!((kv.first >> j0) & 1u)) j0++;
                    std::string ld = dval(oi, op.ridx[j0], "ib" + std::to_string(oi));
                    const std::string cnd = op_cond(op);      // guarded op: factor 1 where the guard fails
                    if (!cnd.empty()) ld = "((" + cnd + ") ? " + ld + " : mk(1.0, 0.0))";
                    if (first) k << "        double2 " << U << " = " << ld << ";\n";
                    else k << "        " << U << " = cmul(" << U << ", " << ld << ");\n";
                    first = false;
                }
                for (int j = 0; j < RA; j++)
                    if ((kv.first >> j) & 1u) fac[j].push_back(U);
            }
            for (int oi : var) {
                const dev::RegOp &op = ops[oi];
                std::map<uint32_t, std::string> sym;
                for (int j = 0; j < RA; j++) {
                    if ((j & op.rcm) != op.rcv) continue;
                    auto it = sym.find(op.ridx[j]);
                    if (it == sym.end()) {
                        const std::string L = "L" + std::to_string(oi) + "_" + std::to_string(op.ridx[j]);
                        const std::string cnd = op_cond(op);
                        k << "        const double2 " << L << " = " << (cnd.empty() ? "" : "(" + cnd + ") ? ")
                          << dval(oi, op.ridx[j], "ib" + std::to_string(oi)) << (cnd.empty() ? "" : " : mk(1.0, 0.0)")
                          << ";\n";
                        it = sym.emplace(op.ridx[j], L).first;
                    }
                    fac[j].push_back(it->second);
                }
            }
            std::map<std::vector<std::string>, std::string> prod;
            int nf = 0;
            for (int j = 0; j < RA; j++) {
                if (fac[j].empty()) continue;
                std::string f = fac[j][0];
                for (size_t q = 1; q < fac[j].size(); q++) {
                    std::vector<std::string> key(fac[j].begin(), fac[j].begin() + q + 1);
                    auto it = prod.find(key);
                    if (it == prod.end()) {
                        const std::string F = "F" + std::to_string(nf++);
                        k << "        const double2 " << F << " = cmul(" << f << ", " << fac[j][q] << ");\n";
                        it = prod.emplace(key, F).first;
                    }
                    f = it->second;
                }
                if (A >= 0 && ((j >> A) & 1)) {        // folded into the butterfly that follows
                    const std::string w = "pw" + std::to_string(pid) + "_" + std::to_string(j);
                    k << "        " << w << " = " << f << ";\n";
                    pend[j] = w;
                } else {
                    k << "        v" << j << " = cmul(" << f << ", v" << j << ");\n";
                }
            }
            k << "      }\n";
        };
        const bool group_on = cfg.group && !var.no_group;
        for (int oi = P.op0; oi < P.op1 && !cfg.skeleton && !vdm; oi++) {
            const WRun *wr = nullptr;
            for (auto &w : wruns)
                if (w.p == (int)p && w.a == oi) wr = &w;
            if (wr) {
                flush_all();
                tail_in_smem = false;
                const int C = 1 << wr->V.size();
                auto ent = [&](int q, const std::string &idx) {      // entry idx of op q's matrix
                    auto cs = cstage.find(q);
                    if (cs != cstage.end()) return "cwa.w[" + std::to_string(cs->second) + "u + " + idx + "]";
                    return "__ldg(blob + " + std::to_string(ops[q].data_off) + "ull + " + idx + ")";
                };
                k << "      { // wide run of " << (wr->b - wr->a) << " ops: per-tile products over " << C << " thread-bit combos\n";
                k << "        const u32 we = threadIdx.x, wr_ = we >> 4, wc_ = we & 15u;\n";
                k << "        bar();      // a previous run's readers are done with the tables\n";
                for (int c = 0; c < C; c++)
                    k << "        wtab[" << c * 257 << "u + we] = (wr_ == wc_) ? mk(1.0, 0.0) : mk(0.0, 0.0);\n";
                k << "        u32 pb = 0u;\n        bar();\n";
                for (int q = wr->a; q < wr->b; q++) {
                    const auto &op = ops[q];
                    if (op.gcm) k << "        if ((gbase & " << u64s(op.gcm) << ") == " << u64s(op.gcv) << ") {\n";
                    else k << "        {\n";
                    k << "          const u32 po = pb * " << C * 257 << "u, pn = (pb ^ 1u) * " << C * 257 << "u;\n";
                    bool any = false;
                    for (int c = 0; c < C; c++) {
                        uint32_t ctb = 0;
                        for (size_t i = 0; i < wr->V.size(); i++)
                            if ((c >> i) & 1) ctb |= 1u << wr->V[i];
                        const bool act = (ctb & op.tcm) == op.tcv;
                        if (act) {
                            if (!any) {      // this thread's matrix row, shared by the combos
                                for (int kk = 0; kk < 16; kk++)
                                    k << "          const double2 u" << kk << " = " << ent(q, "wr_ * 16u + " + std::to_string(kk) + "u") << ";\n";
                                any = true;
                            }
                            k << "          { double ax = 0.0, ay = 0.0;";
                            for (int kk = 0; kk < 16; kk++)
                                k << " { const double2 t = wtab[po + " << c * 257 + kk * 16 << "u + wc_]; ax = fma(u" << kk
                                  << ".x, t.x, ax); ax = fma(-u" << kk << ".y, t.y, ax); ay = fma(u" << kk << ".x, t.y, ay); ay = fma(u"
                                  << kk << ".y, t.x, ay); }";
                            k << " wtab[pn + " << c * 257 << "u + we] = mk(ax, ay); }\n";
                        } else {
                            // (a value copy: a bare wtab[] = wtab[] would assign the shared-memory proxy itself)
                            k << "          wtab[pn + " << c * 257 << "u + we] = (double2)wtab[po + " << c * 257 << "u + we];\n";
                        }
                    }
                    k << "          pb ^= 1u;\n          bar();\n        }\n";
                }
                // apply this thread's product (combo from its thread bits), rows to its own smem slots
                k << "        const u32 mc = 0u";
                for (size_t i = 0; i < wr->V.size(); i++) k << " | (((tb >> " << wr->V[i] << ") & 1u) << " << i << ")";
                k << ";\n        const u32 pm = pb * " << C * 257 << "u + mc * 257u;\n";
                k << "        #pragma unroll 1\n        for (u32 r = 0; r < 16u; r++) { double ax = 0.0, ay = 0.0;";
                for (int kk = 0; kk < 16; kk++)
                    k << " { const double2 w = wtab[pm + r * 16u + " << kk << "u]; ax = fma(w.x, v" << kk << ".x, ax); ax = fma(-w.y, v"
                      << kk << ".y, ax); ay = fma(w.x, v" << kk << ".y, ay); ay = fma(w.y, v" << kk << ".x, ay); }";
                k << " const u32 slot = " << rd[0] << "u";
                for (int i = 0; i < 4; i++) k << " | ((r >> " << i << ") & 1u) << " << P.R[i];
                k << "; cur[swz(tb | slot)] = mk(ax, ay); }\n";
                for (int r = 0; r < 16; r++) k << "        v" << r << " = " << sref(rd[r]) << ";\n";
                // the tables are rewritten by the next run / tile only after a barrier: the end of this
                // phase (or tile) has one, and a following run starts with one after its init
                k << "      }\n";
                oi = wr->b - 1;
                continue;
            }
            const DRun *run = nullptr;
            for (auto &dr : druns)
                if (dr.p == (int)p && oi >= dr.a && oi < dr.b) run = &dr;
            if (run) {
                if (oi == run->a) flush_all();
                if (oi == run->a) {      // the whole run: one shared lookup + one complex multiply per slot
                    const int nv = (int)run->V.size();
                    k << "      { const u32 bt = 0u";
                    for (int i = 0; i < nv; i++)
                        if (std::find(P.R, P.R + RB, run->V[i]) == P.R + RB)
                            k << " | (((tb >> " << run->V[i] << ") & 1u) << " << i << ")";
                    k << "; // diagonal run of " << (run->b - run->a) << " ops\n";
                    for (int j = 0; j < RA; j++) {
                        bool touched = false;      // slots outside every op's register controls keep factor 1
                        for (int q = run->a; q < run->b; q++)
                            if ((j & ops[q].rcm) == ops[q].rcv) touched = true;
                        if (!touched) continue;
                        int cj = 0;
                        for (int i = 0; i < nv; i++)
                            for (int r = 0; r < RB; r++)
                                if (P.R[r] == run->V[i] && ((j >> r) & 1)) cj |= 1 << i;
                        k << "        v" << j << " = cmul(dsub[" << run->off << " + (bt | " << cj << "u)], v" << j << ");\n";
                    }
                    k << "      }\n";
                }
                continue;
            }
            if (group_on && ops[oi].kind == 1) {
                auto in_run = [&](int q) {
                    for (auto &dr : druns)
                        if (dr.p == (int)p && q >= dr.a && q < dr.b) return true;
                    return false;
                };
                int oj = oi;
                while (oj < P.op1 && ops[oj].kind == 1 && !in_run(oj)) oj++;
                std::vector<int> G, C;
                for (int q = oi; q < oj; q++) G.push_back(q);
                if (G.size() >= 2) {
                    emit_group(G, bfly_bit(oj));
                    for (int q : C) emit_single(q);
                    oi = oj - 1;
                    continue;
                }
            }
            emit_single(oi);
        }
        flush_all();
        // hoisted sub-table build for the next phase (or the next tile's phase 0) after this phase's
        // registers are stored (they are dead: no extra register pressure), before the barrier
        auto hoisted = [&] {
            if (!hoist) return;
            if (p + 1 < nph) emit_pre(p + 1, "gbase");
            else {
                k << "      if (tile + gridDim.x < n_tiles) {\n";
                emit_pre(0, "rank_base | tile_base(tile + gridDim.x)");
                k << "      }\n";
            }
        };
        if (p + 1 == ph.size() && dout) {
            k << "      double2 *gout = psi + (base | pd_out);\n";
            if (red) k << "      double r0 = 0.0, r1 = 0.0;\n";
            for (int j = 0; j < RA; j++) {
                if ((uint32_t)rd[j] & a.zstore) continue;          // still known zero: not written
                const std::string zc = a.zstore ? "if (!(tb & " + std::to_string(a.zstore) + "u)) " : std::string();
                k << "      " << zc << "__stcs(gout + " << u64s(phys_slot(P, j)) << ", v" << j << ");\n";
                if (red)      // slot offsets with the bit set go to r1; the rest follow (base | pd_out)'s bit
                    k << "      " << zc << ((phys_slot(P, j) >> a.red) & 1 ? "r1" : "r0") << " = fma(v" << j << ".x, v"
                      << j << ".x, fma(v" << j << ".y, v" << j << ".y, " << ((phys_slot(P, j) >> a.red) & 1 ? "r1" : "r0")
                      << "));\n";
            }
            if (red)
                k << "      if (((base | pd_out) >> " << rbs << ") & 1ull) q1 += r0 + r1; else { q0 += r0; q1 += r1; }\n";
            hoisted();
            k << "    }\n";
        } else {
            if (!tail_in_smem)
                for (int j = 0; j < RA; j++) k << "      " << sref(rd[j]) << " = v" << j << ";\n";
            hoisted();
            k << "      bar();\n    }\n";
        }
    }
    if (!dout) {
        const std::string zc = a.zstore ? "if (!(u & " + std::to_string(a.zstore) + "u)) " : std::string();
        if (red)
            k << "    for (u32 u = threadIdx.x; u < NT; u += " << NTHR << ") " << zc
              << "{ const u64 ad = addr(base, u); const double2 x = cur[swz(u)]; psi[ad] = x; const double w = "
                 "fma(x.x, x.x, x.y * x.y); if ((ad >> "
              << rbs << ") & 1ull) q1 += w; else q0 += w; }\n";
        else
            k << "    for (u32 u = threadIdx.x; u < NT; u += " << NTHR << ") " << zc << "psi[addr(base, u)] = cur[swz(u)];\n";
    }
    // one barrier per tile: the next tile's first shared-memory write (cp.async, phase-0 stores,
    // diagonal sub-tables) must not overtake a slower warp still reading this tile's last phase
    k << "    bar();\n  }\n  cp_async_wait0();\n";
    if (red) {      // every thread left the loop after the last tile's barrier: the tile buffer is free
        const int g = NTHR >= 16 ? 16 : NTHR;
        k << "  buf0[threadIdx.x] = mk(q0, q1);\n  bar();\n";
        k << "  if (threadIdx.x < " << g << "u) { double s0 = 0.0, s1 = 0.0; for (u32 i = threadIdx.x; i < " << NTHR
          << "u; i += " << g << "u) { const double2 t = buf0[i]; s0 += t.x; s1 += t.y; } buf0[" << NTHR
          << "u + threadIdx.x] = mk(s0, s1); }\n  bar();\n";
        k << "  if (threadIdx.x == 0) { double s0 = 0.0, s1 = 0.0; for (u32 i = 0; i < " << g << "u; i++) { const double2 t = buf0["
          << NTHR << "u + i]; s0 += t.x; s1 += t.y; } red[2ull * blockIdx.x] = s0; red[2ull * blockIdx.x + 1ull] = s1; }\n";
    }
    k << "}\n";
    return k.str();
}

// ---------------------------------------------------------------- compile ----
namespace {
// One compiled + loaded tile kernel per distinct source text. The thread that inserts an entry owns
// its compilation; every other thread that finds it (a concurrent program creation on another
// thread, or the same source twice in one program) waits on `ready` until the owner has published
// lib/kern/err. Only the owner erases a failed entry (so a later call can retry).
struct CacheEntry {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    std::string err;
    std::promise<void> done;
    std::shared_future<void> ready;
    CacheEntry() : ready(done.get_future().share()) {}
};
std::mutex g_mu;
std::map<std::string, std::shared_ptr<CacheEntry>> g_cache;

std::vector<char> compile_cubin(const std::string &src, std::string &err, int *spill = nullptr) {
    Nvrtc &n = nvrtc();
    nvrtcProgram_t prog = nullptr;
    const std::string full = std::string(kPrelude) + src;
    // developer aid (HHLSV_JIT_DUMP=dir): keep source + cubin, named by a hash of the source; the
    // source path is the program name, so -lineinfo maps SASS to it (ncu --import-source)
    std::string stem;
    if (const char *dir = getenv("HHLSV_JIT_DUMP")) {
        stem = std::string(dir) + "/" + jit_source_tag(src);
        if (FILE *f = fopen((stem + ".cu").c_str(), "w")) {
            fwrite(full.data(), 1, full.size(), f);
            fclose(f);
        }
    }
    if (n.create(&prog, full.c_str(), stem.empty() ? "hhlsv_tile.cu" : (stem + ".cu").c_str(), 0, nullptr, nullptr)) {
        err = "nvrtcCreateProgram failed";
        return {};
    }
    // Shared memory is addressed through explicit 32-bit shared-window addresses (lds/sts in the
    // prelude): with NVRTC's default 64-bit shared-pointer arithmetic, ptxas -O2/-O3 miscompiled
    // some tile kernels into illegal-address faults (source clean under host emulation with
    // ASan/UBSan, scripts/jit_emulate.py; same PTX fine at -O1).
    std::vector<const char *> opts = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-Xptxas=-v", "-Xptxas=-O3"};
    const JitConfig &cfg = jit_config();
    if (!cfg.ptxas_opt.empty()) opts.back() = cfg.ptxas_opt.c_str();
    if (cfg.smem_clobber) opts.push_back("-DHHLSV_SMEM_CLOBBER");
    int rc = n.compile(prog, (int)opts.size(), opts.data());
    if (rc) {
        size_t ls = 0;
        n.logSize(prog, &ls);
        std::string log(ls, '\0');
        n.log(prog, &log[0]);
        err = std::string("NVRTC: ") + n.errStr(rc) + "\n" + log.substr(0, 2000);
        n.destroy(&prog);
        return {};
    }
    if (spill) {        // ptxas -v: "N bytes stack frame, S bytes spill stores, L bytes spill loads"
        size_t ls = 0;
        n.logSize(prog, &ls);
        std::string log(ls, '\0');
        if (ls) n.log(prog, &log[0]);
        *spill = 0;
        const size_t at = log.find(" bytes spill stores");
        if (at != std::string::npos) {
            size_t b = log.rfind(',', at);
            b = (b == std::string::npos) ? 0 : b + 1;
            *spill = std::atoi(log.c_str() + b);
        }
    }
    size_t cs = 0;
    n.cubinSize(prog, &cs);
    std::vector<char> cubin(cs);
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    if (!stem.empty()) {
        if (FILE *f = fopen((stem + ".cubin").c_str(), "wb")) {
            fwrite(cubin.data(), 1, cubin.size(), f);
            fclose(f);
        }
    }
    return cubin;
}
// Cubins compiled ahead of jit_build (spill probing): source -> (cubin, spill bytes). jit_build and
// jit_compile_only take their entry (a probed pass is compiled once).
std::mutex g_cub_mu;
std::map<std::string, std::pair<std::vector<char>, int>> g_cubins;
std::map<size_t, int> g_spill;       // hash of the source -> ptxas spill-store bytes (kept for the process)

std::vector<char> take_or_compile(const std::string &src, std::string &err) {
    {
        std::lock_guard<std::mutex> lk(g_cub_mu);
        auto it = g_cubins.find(src);
        if (it != g_cubins.end()) {
            std::vector<char> c = std::move(it->second.first);
            g_cubins.erase(it);
            if (!c.empty()) return c;
        }
    }
    return compile_cubin(src, err);
}
}  // namespace

bool jit_spill_cached(const std::string &src, int *spill) {
    std::lock_guard<std::mutex> lk(g_cub_mu);
    auto it = g_spill.find(std::hash<std::string>()(src));
    if (it == g_spill.end()) return false;
    *spill = it->second;
    return true;
}

int jit_spill_bytes(const std::string &src) {
    int known = 0;
    if (jit_spill_cached(src, &known)) return known;
    if (!nvrtc().ok) return -1;
    std::string err;
    int spill = 0;
    std::vector<char> c = compile_cubin(src, err, &spill);
    if (c.empty()) return -1;
    std::lock_guard<std::mutex> lk(g_cub_mu);
    g_spill[std::hash<std::string>()(src)] = spill;
    g_cubins[src] = {std::move(c), spill};      // taken by the jit_build that loads it
    return spill;
}

std::string jit_source_tag(const std::string &src) {
    char hx[32];
    snprintf(hx, sizeof hx, "%016zx", std::hash<std::string>()(std::string(kPrelude) + src));
    return std::string("tile_") + hx;
}

std::vector<char> jit_compile_only(const std::string &src, std::string &err) {
    if (!nvrtc().ok) {
        err = nvrtc().why;
        return {};
    }
    return take_or_compile(src, err);
}

void jit_build(std::vector<JitPass> &passes) {
    if (!nvrtc().ok) fail(SV_E_CUDA, "tile JIT unavailable: " + nvrtc().why);
    // compile the passes not yet in the cache in parallel (NVRTC programs are independent)
    std::vector<std::shared_ptr<CacheEntry>> ents(passes.size());
    std::vector<size_t> todo;       // entries this call owns
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (size_t i = 0; i < passes.size(); i++) {
            auto it = g_cache.find(passes[i].src);
            if (it != g_cache.end()) {
                ents[i] = it->second;
            } else {
                ents[i] = std::make_shared<CacheEntry>();
                g_cache[passes[i].src] = ents[i];
                todo.push_back(i);
            }
        }
    }
    std::vector<std::vector<char>> cubins(passes.size());
    std::vector<std::thread> th;
    for (size_t i : todo)
        th.emplace_back([&, i] { cubins[i] = take_or_compile(passes[i].src, ents[i]->err); });
    for (auto &t : th) t.join();
    for (size_t i : todo) {
        CacheEntry &e = *ents[i];
        if (!cubins[i].empty()) {
            cudaError_t rc = cudaLibraryLoadData(&e.lib, cubins[i].data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
            if (rc == cudaSuccess) rc = cudaLibraryGetKernel(&e.kern, e.lib, passes[i].name.c_str());
            if (rc != cudaSuccess) {
                e.kern = nullptr;
                e.err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(rc);
            }
        }
        if (!e.kern) {               // owner: drop the failed entry so a later build can retry
            std::lock_guard<std::mutex> lk(g_mu);
            auto it = g_cache.find(passes[i].src);
            if (it != g_cache.end() && it->second == ents[i]) g_cache.erase(it);
        }
        e.done.set_value();          // publishes lib / kern / err to every waiter
    }
    for (size_t i = 0; i < passes.size(); i++) {
        ents[i]->ready.wait();
        if (!ents[i]->kern) fail(SV_E_CUDA, "tile JIT failed: " + ents[i]->err);
        passes[i].kern = ents[i]->kern;
    }
}

size_t jit_smem_bytes(int T, size_t total) {
    (void)T;
    return total;
}

cudaError_t jit_launch(const JitPass &p, double2 *psi, const double2 *blob, uint64_t n_tiles, uint64_t rank_base,
                       int T, cudaStream_t s, uint64_t tile0) {
    const int threads = p.nthr;
    const size_t smem = jit_smem_bytes(T, p.smem_extra);
    const void *f = reinterpret_cast<const void *>(p.kern);
    cudaError_t e = cudaSuccess;
    if (p.per_sm == 0) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem);
        if (e != cudaSuccess) return e;
        p.per_sm = per_sm < 1 ? 1 : per_sm;
        int dev = 0, sms = 0;
        e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        p.sms = sms;                 // 148 on the B200: persistent grid = SMs x resident CTAs
    }
    if (tile0 >= n_tiles) return cudaSuccess;
    uint64_t grid = (uint64_t)p.sms * p.per_sm;
    if (grid > n_tiles - tile0) grid = n_tiles - tile0;
    double *red = p.red;
    void *args[7] = {&psi, (void *)&blob, &n_tiles, &rank_base, &tile0};
    int na = 5;
    if (red) args[na++] = &red;
    args[na++] = (void *)p.cwvals.data();
    return cudaLaunchKernel(f, dim3((unsigned)grid), dim3(threads), args, smem, s);
}

uint64_t jit_grid(const JitPass &p, uint64_t n_tiles) {
    const uint64_t g = (uint64_t)p.sms * p.per_sm;
    return g < n_tiles ? g : n_tiles;
}

}  // namespace hhlsv
