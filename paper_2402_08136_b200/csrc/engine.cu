// Device state, resident programs and readout.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>

#include <map>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "engine.h"

namespace hhlsv {

void cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) fail(SV_E_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(SV_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static void nccl_check(int rc, const char *what) {
    if (rc) fail(SV_E_NCCL, std::string(what) + ": " + nccl_last_error());
}

// ------------------------------------------------------------------ state ----
// State buffers come from a stream-ordered memory pool OWNED BY THE LIBRARY (one per device, never
// the process-wide default pool, so other allocators in the process -- e.g. torch -- are not
// starved) with an unbounded release threshold: freeing a 16 GiB state and creating the next one
// (hhl_solve called repeatedly) reuses the pool instead of unmapping/remapping pages (measured on the
// B200: trimming after every solve makes the next 16 GiB allocation cost ~4.7 s, a partial trim ~5 ms).
// The memory stays cached for the next state; sv_trim_memory() releases it, and state_create trims
// before reporting OOM (so the cache never makes a state fail to fit).
namespace {
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};
int g_live_states = 0;
}  // namespace

void pool_trim(int device, size_t keep) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (int d = 0; d < 64; d++)
        if (g_pools[d] && (device < 0 || d == device)) cudaMemPoolTrimTo(g_pools[d], keep);
}

static cudaMemPool_t lib_pool(int device) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (device < 0 || device >= 64) fail(SV_E_ARG, "device index out of range");
    if (!g_pools[device]) {
        cudaMemPoolProps pr{};
        pr.allocType = cudaMemAllocationTypePinned;
        pr.handleTypes = cudaMemHandleTypeNone;
        pr.location.type = cudaMemLocationTypeDevice;
        pr.location.id = device;
        cuda_check(cudaMemPoolCreate(&g_pools[device], &pr), "cudaMemPoolCreate");
        uint64_t thr = UINT64_MAX;
        cuda_check(cudaMemPoolSetAttribute(g_pools[device], cudaMemPoolAttrReleaseThreshold, &thr), "pool threshold");
    }
    return g_pools[device];
}

// Bytes the library pool of `device` holds reserved but not in use (reusable by the next state).
static size_t pool_slack(int device) {
    cudaMemPool_t pool = lib_pool(device);
    uint64_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    return reserved > used ? (size_t)(reserved - used) : 0;
}

static cudaError_t state_alloc(void **p, size_t bytes, cudaStream_t s, int device) {
    cudaError_t e = cudaMallocFromPoolAsync(p, bytes, lib_pool(device), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e;
}
static void state_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// Small per-state / per-program device buffers also come from the stream-ordered pool: a plain
// cudaFree is device-synchronising and (measured) can stall for ~0.2 s when the driver trims
// memory after a 16 GiB state was released; pool frees are stream-ordered and cheap.
static cudaError_t pool_malloc(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    return state_alloc(p, bytes, s, dev);
}
// Stream-ordered allocation without the synchronisation (the caller synchronises once for a batch).
static cudaError_t pool_malloc_nosync(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    return cudaMallocFromPoolAsync(p, bytes, lib_pool(dev), s);
}
static void pool_free(void *p, cudaStream_t s) { state_free(p, s); }

sv_state *state_create(int n, const sv_dist *dist, cudaStream_t stream, bool zero_init) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        fail(SV_E_CUDA, "no CUDA device: this library has no CPU fallback");
    }
    int world = 1, rank = 0, device = -1;
    if (dist) {
        world = dist->world;
        rank = dist->rank;
        device = dist->device;
        if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world)
            fail(SV_E_ARG, "sv_dist: world must be a power of two and 0 <= rank < world");
    }
    const bool virt = world > 1 && !dist->nccl_id;
    int g = 0;
    while ((1 << g) < world) g++;
    if (n < 1 || n - g < 1 || n > 62) fail(SV_E_ARG, "n_qubits out of range");
    if (device >= 0) cuda_check(cudaSetDevice(device), "cudaSetDevice");
    else cuda_check(cudaGetDevice(&device), "cudaGetDevice");
    std::unique_ptr<sv_state> sv(new sv_state());
    sv->n = n;
    sv->g = g;
    sv->nloc = n - g;
    sv->world = world;
    sv->rank = rank;
    sv->device = device;
    sv->stream = stream;
    sv->phys.resize(n);
    std::iota(sv->phys.begin(), sv->phys.end(), 0);
    const size_t bytes = sizeof(double2) << sv->nloc;
    // Fits in what the library pool already holds free (a repeated solve): no device-memory query
    // (cudaMemGetInfo measured 0.1-97 ms on the B200 while another 16 GiB state is resident).
    size_t freeb = pool_slack(device), totb = 0;
    if (bytes * (virt ? world : 1) > freeb) {
        cuda_check(cudaMemGetInfo(&freeb, &totb), "cudaMemGetInfo");
        freeb += pool_slack(device);     // reserved by the library pool but free for reuse
    }
    if (bytes * (virt ? world : 1) > freeb) {   // release cached pool memory, then decide
        cuda_check(cudaDeviceSynchronize(), "sync before trim");
        pool_trim(device, 0);
        cuda_check(cudaMemGetInfo(&freeb, &totb), "cudaMemGetInfo");
        freeb += pool_slack(device);
        if (bytes * (virt ? world : 1) > freeb) fail(SV_E_OOM, "state does not fit in device memory");
    }

    if (virt) {
        sv->vworld = world;
        sv->world = 1;
        for (int r = 0; r < world; r++) {
            std::unique_ptr<sv_state> v(new sv_state());
            v->n = n;
            v->g = g;
            v->nloc = n - g;
            v->world = 1;
            v->rank = r;
            v->device = device;
            v->stream = stream;
            v->phys = sv->phys;
            cuda_check(state_alloc((void **)&v->psi, bytes, stream, device), "alloc(virtual shard)");
            v->red_len = dev::kRedBlocks;
            cuda_check(pool_malloc((void **)&v->d_red, sizeof(double) * v->red_len, stream), "cudaMalloc(red)");
            cuda_check(pool_malloc((void **)&v->d_scalar, sizeof(double) * 8, stream), "cudaMalloc(scalar)");
            sv->views.push_back(v.release());
        }
        sv->psi = sv->views[0]->psi;
    } else {
        prof_mark("    state: size check");
        cuda_check(state_alloc((void **)&sv->psi, bytes, stream, device), "alloc(state)");
        prof_mark("    state: alloc");
    }
    sv->red_len = dev::kRedBlocks;
    cuda_check(pool_malloc_nosync((void **)&sv->d_red, sizeof(double) * sv->red_len, stream), "cudaMalloc(red)");
    cuda_check(pool_malloc_nosync((void **)&sv->d_scalar, sizeof(double) * 8, stream), "cudaMalloc(scalar)");
    cuda_check(cudaStreamSynchronize(stream), "alloc sync");
    if (world > 1 && !virt) nccl_check(nccl_init(sv->comm, world, rank, dist->nccl_id), "ncclCommInitRank");
    if (zero_init) state_reset(sv.get());
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        g_live_states++;
    }
    return sv.release();
}

static void destroy_impl(sv_state *sv, bool top);
void state_destroy(sv_state *sv) { destroy_impl(sv, true); }

static void destroy_impl(sv_state *sv, bool top) {
    if (!sv) return;
    cudaStreamSynchronize(sv->stream);
    if (sv->vworld > 1) {
        for (auto *v : sv->views) destroy_impl(v, false);
        sv->views.clear();
        sv->psi = nullptr;
    }
    state_free(sv->psi, sv->stream);
    pool_free(sv->d_red, sv->stream);
    pool_free(sv->d_scalar, sv->stream);
    pool_free(sv->d_io, sv->stream);
    pool_free(sv->d_xsend, sv->stream);
    pool_free(sv->d_xrecv, sv->stream);
    nccl_destroy(sv->comm);
    if (sv->comm_stream) cudaStreamDestroy(sv->comm_stream);
    if (sv->ev_a) cudaEventDestroy(sv->ev_a);
    if (sv->ev_b) cudaEventDestroy(sv->ev_b);
    const int device = sv->device;
    cudaStreamSynchronize(sv->stream);
    delete sv;
    if (!top) return;
    (void)device;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (--g_live_states < 0) g_live_states = 0;
    // the pool keeps its memory for the next state (measured: even a trim that keeps one state's worth
    // costs the next 16 GiB allocation ~5 ms of re-mapping); it is released when a new state would not
    // fit otherwise (state_create) or by sv_trim_memory
}

void state_reset(sv_state *sv) {
    std::iota(sv->phys.begin(), sv->phys.end(), 0);
    if (sv->vworld > 1) {
        for (auto *v : sv->views) state_reset(v);
        return;
    }
    cuda_check(dev::launch_zero_init(sv->psi, sv->local_amps(), sv->rank == 0, sv->stream), "init zero");
}

static void ensure_io(sv_state *sv, size_t n2) {
    if (sv->io_len >= n2) return;
    pool_free(sv->d_io, sv->stream);
    sv->d_io = nullptr;
    sv->io_len = 0;
    cuda_check(pool_malloc((void **)&sv->d_io, sizeof(double2) * n2, sv->stream), "cudaMalloc(io)");
    sv->io_len = n2;
}

static void ensure_red(sv_state *sv, size_t n) {
    if (sv->red_len >= n) return;
    pool_free(sv->d_red, sv->stream);
    sv->d_red = nullptr;
    cuda_check(pool_malloc((void **)&sv->d_red, sizeof(double) * n, sv->stream), "cudaMalloc(red)");
    sv->red_len = n;
}

// --------------------------------------------------------------- exchange ----
// Multi-qubit exchange: swap the values of physical global bits G[i] with local bits
// L[i]. With the pairs ordered by ascending L, bit i of a slot pattern p <-> L[i]. Rank r holds, in
// slot p (its elements whose L bits equal p), amplitudes that belong to rank peer(r, p) = r with its
// G bits set to p; they land there in slot own(r) = r's G pattern. So rank r sends slot p to
// peer(r, p) and receives slot p from the same peer: an all-to-all among the 2^k ranks that share r's
// other global bits, (1 - 2^-k) of the shard each way (k = 1: the pairwise half-swap). Chunked
// (<= 2^24 amplitudes per slot per round); when L are the top k local bits every slot is contiguous
// and is sent straight from the state (no pack kernel).
struct XPlan {
    int k = 0;
    std::vector<int> Ls, Gs;
    uint32_t own = 0;
    uint64_t slot = 0;
    bool top = false;
};
static XPlan xplan(const sv_state *sv, int rank, const std::vector<int> &G, const std::vector<int> &L) {
    XPlan x;
    x.k = (int)G.size();
    std::vector<std::pair<int, int>> pr;
    for (int i = 0; i < x.k; i++) pr.push_back({L[i], G[i]});
    std::sort(pr.begin(), pr.end());
    for (auto &q : pr) {
        x.Ls.push_back(q.first);
        x.Gs.push_back(q.second);
    }
    for (int i = 0; i < x.k; i++) x.own |= (uint32_t)((rank >> (x.Gs[i] - sv->nloc)) & 1) << i;
    x.slot = sv->local_amps() >> x.k;
    x.top = true;
    for (int i = 0; i < x.k; i++) x.top &= x.Ls[i] == sv->nloc - x.k + i;
    return x;
}
static int xpeer(const sv_state *sv, const XPlan &x, int rank, uint32_t p) {
    int r = rank;
    for (int i = 0; i < x.k; i++) {
        const int gb = x.Gs[i] - sv->nloc;
        r = (r & ~(1 << gb)) | (int)(((p >> i) & 1u) << gb);
    }
    return r;
}
static uint64_t xchunk(const XPlan &x) { return std::min<uint64_t>(x.slot, 1ull << 24); }

static void ensure_xbuf(sv_state *sv, size_t n) {
    if (sv->x_len >= n) return;
    pool_free(sv->d_xsend, sv->stream);
    pool_free(sv->d_xrecv, sv->stream);
    sv->d_xsend = sv->d_xrecv = nullptr;
    sv->x_len = 0;
    cuda_check(pool_malloc((void **)&sv->d_xsend, sizeof(double2) * n, sv->stream), "cudaMalloc(xsend)");
    cuda_check(pool_malloc((void **)&sv->d_xrecv, sizeof(double2) * n, sv->stream), "cudaMalloc(xrecv)");
    sv->x_len = n;
}

static void exchange(sv_state *sv, const std::vector<int> &G, const std::vector<int> &L) {
    const XPlan x = xplan(sv, sv->rank, G, L);
    const uint32_t np = (1u << x.k) - 1;
    const uint64_t C = xchunk(x);
    ensure_xbuf(sv, (size_t)np * C);
    std::vector<const double *> sb(np);
    std::vector<double *> rb(np);
    std::vector<int> peers(np);
    for (uint64_t off = 0; off < x.slot; off += C) {
        const uint64_t cnt = std::min(C, x.slot - off);
        uint32_t i = 0;
        for (uint32_t p = 0; p <= np; p++) {
            if (p == x.own) continue;
            peers[i] = xpeer(sv, x, sv->rank, p);
            rb[i] = (double *)(sv->d_xrecv + (size_t)i * C);
            if (x.top) {
                sb[i] = (const double *)(sv->psi + (uint64_t)p * x.slot + off);
            } else {
                cuda_check(dev::launch_pack_multi(sv->psi, sv->d_xsend + (size_t)i * C, x.Ls.data(), x.k, p, off, cnt,
                                                  sv->stream),
                           "exchange pack");
                sb[i] = (const double *)(sv->d_xsend + (size_t)i * C);
            }
            i++;
        }
        nccl_check(nccl_alltoall_pairs(sv->comm, sb.data(), rb.data(), peers.data(), (int)np, 2 * cnt, sv->stream),
                   "exchange all-to-all");
        i = 0;
        for (uint32_t p = 0; p <= np; p++) {
            if (p == x.own) continue;
            if (x.top)
                cuda_check(cudaMemcpyAsync(sv->psi + (uint64_t)p * x.slot + off, sv->d_xrecv + (size_t)i * C,
                                           sizeof(double2) * cnt, cudaMemcpyDeviceToDevice, sv->stream),
                           "exchange copy");
            else
                cuda_check(dev::launch_unpack_multi(sv->psi, sv->d_xrecv + (size_t)i * C, x.Ls.data(), x.k, p, off, cnt,
                                                    sv->stream),
                           "exchange unpack");
            i++;
        }
    }
}

// Virtual sharding: the same exchange between the in-process shards (device copies): for every
// rank r and pattern p != own(r) with s = peer(r, p) > r, swap r's slot p with s's slot own(r).
static void virtual_exchange(sv_state *sv, const std::vector<int> &G, const std::vector<int> &L) {
    const sv_state *v0 = sv->views[0];
    const XPlan x0 = xplan(v0, 0, G, L);
    const uint64_t C = xchunk(x0);
    ensure_xbuf(sv, C);
    for (int r = 0; r < sv->vworld; r++) {
        const XPlan xr = xplan(v0, r, G, L);
        for (uint32_t p = 0; p < (1u << xr.k); p++) {
            if (p == xr.own) continue;
            const int s = xpeer(v0, xr, r, p);
            if (s < r) continue;
            sv_state *A = sv->views[r], *B = sv->views[s];
            for (uint64_t off = 0; off < xr.slot; off += C) {
                const uint64_t cnt = std::min(C, xr.slot - off);
                cuda_check(dev::launch_pack_multi(A->psi, sv->d_xsend, xr.Ls.data(), xr.k, p, off, cnt, sv->stream), "vpack");
                cuda_check(dev::launch_pack_multi(B->psi, sv->d_xrecv, xr.Ls.data(), xr.k, xr.own, off, cnt, sv->stream),
                           "vpack");
                cuda_check(dev::launch_unpack_multi(A->psi, sv->d_xrecv, xr.Ls.data(), xr.k, p, off, cnt, sv->stream),
                           "vunpack");
                cuda_check(dev::launch_unpack_multi(B->psi, sv->d_xsend, xr.Ls.data(), xr.k, xr.own, off, cnt, sv->stream),
                           "vunpack");
            }
        }
    }
}

// ---------------------------------------------------------------- program ----
static int popc64(uint64_t x) { return __builtin_popcountll(x); }

// FP64 flops per amplitude a register-phase op executes (complex MAC = 8, real x complex = 4,
// complex multiply = 6, butterfly/scale = 2, reciprocal rotation ~6 per amplitude), times the
// fraction of amplitudes its controls / control-like diagonal bits select.
double regop_flops(const dev::RegOp &r) {
    const double sel = std::ldexp(1.0, -(popc64((uint64_t)r.rcm) + popc64(r.tcm) + popc64(r.gcm)));
    switch (r.kind) {
        case 0: {
            const int K = popc64((uint64_t)r.mask);
            return (r.is_signed ? 4.0 : 8.0) * std::ldexp(1.0, K) * sel;
        }
        case 1: return 6.0 * sel;
        case 2: return 6.0;
        default: return 2.0;
    }
}

static int index_in(const std::vector<int> &v, int x) {
    auto it = std::find(v.begin(), v.end(), x);
    return it == v.end() ? -1 : (int)(it - v.begin());
}

// Product-state init (+ folded leading diagonals): every factor is a table over its own bits.
// Factors whose entries are all equal (e.g. H|0> on every clock qubit) only scale the state: their
// value joins the global scale. The rest are grouped into <= 4 group tables of <= 14 index bits
// (L2-resident), each entry the product of its members, so the init does <= 4 lookups and 3
// complex products per amplitude; amplitudes with a bit no factor covers set are 0.
struct ProductPlan {
    uint64_t zero_mask = 0;
    std::vector<std::vector<int>> bits;      // per group: physical bits, ascending (table bit j <- bits[j])
    std::vector<std::vector<cplx>> tabs;
};

static ProductPlan plan_product(const sv_state *sv, const Step &st, double scale) {
    std::vector<const ProductFactor *> fs;
    uint64_t covered = 0;
    cplx cscale(scale, 0.0);
    for (auto &f : st.factors) {
        if (!f.diag)
            for (int q : f.qubits) covered |= 1ull << q;
        bool uniform = true;
        for (auto &z : f.vec) uniform &= z == f.vec[0];
        if (uniform) {
            cscale *= f.vec[0];
            continue;
        }
        fs.push_back(&f);
    }
    std::stable_sort(fs.begin(), fs.end(), [](const ProductFactor *a, const ProductFactor *b) {
        if (a->diag != b->diag) return !a->diag;
        return *std::min_element(a->qubits.begin(), a->qubits.end()) <
               *std::min_element(b->qubits.begin(), b->qubits.end());
    });
    struct Group {
        std::vector<int> bits;
        std::vector<const ProductFactor *> mem;
    };
    std::vector<Group> groups;
    for (auto *f : fs) {
        int best = -1, best_ov = -1;
        size_t best_u = 0;
        for (size_t gi = 0; gi < groups.size(); gi++) {
            std::vector<int> u = groups[gi].bits;
            int ov = 0;
            for (int q : f->qubits) {
                if (std::find(u.begin(), u.end(), q) == u.end()) u.push_back(q);
                else ov++;
            }
            if (u.size() > 14) continue;
            if (ov > best_ov || (ov == best_ov && u.size() < best_u)) {
                best = (int)gi;
                best_ov = ov;
                best_u = u.size();
            }
        }
        if (best < 0) {
            if (groups.size() == 4) fail(SV_E_ARG, "product initialisation needs more than 4 group tables");
            groups.push_back({});
            best = (int)groups.size() - 1;
        }
        for (int q : f->qubits)
            if (std::find(groups[best].bits.begin(), groups[best].bits.end(), q) == groups[best].bits.end())
                groups[best].bits.push_back(q);
        groups[best].mem.push_back(f);
    }
    if (groups.empty()) groups.push_back({});     // a single scale entry
    ProductPlan pp;
    const uint64_t all = sv->n >= 64 ? ~0ull : ((1ull << sv->n) - 1ull);
    pp.zero_mask = all & ~covered;
    for (size_t gi = 0; gi < groups.size(); gi++) {
        Group &G = groups[gi];
        std::sort(G.bits.begin(), G.bits.end());
        const size_t nb = G.bits.size();
        std::vector<cplx> tab((size_t)1 << nb);
        std::vector<std::vector<int>> pos(G.mem.size());
        for (size_t m = 0; m < G.mem.size(); m++)
            for (int q : G.mem[m]->qubits)
                pos[m].push_back((int)(std::find(G.bits.begin(), G.bits.end(), q) - G.bits.begin()));
        for (size_t x = 0; x < tab.size(); x++) {
            cplx v(1.0, 0.0);
            for (size_t m = 0; m < G.mem.size(); m++) {
                size_t idx = 0;
                for (size_t j = 0; j < pos[m].size(); j++)
                    if ((x >> pos[m][j]) & 1) idx |= (size_t)1 << j;
                v *= G.mem[m]->vec[idx];
            }
            tab[x] = gi == 0 ? v * cscale : v;
        }
        pp.bits.push_back(G.bits);
        pp.tabs.push_back(std::move(tab));
    }
    return pp;
}

static void build_product(sv_state *sv, sv_program *p, const Step &st, LaunchRec &rec, double scale) {
    ProductPlan pp = plan_product(sv, st, scale);
    dev::ProductArgs &a = rec.prod;
    a.psi = sv->psi;
    a.n_amps = sv->local_amps();
    a.rank_base = (uint64_t)sv->rank << sv->nloc;
    a.zero_mask = pp.zero_mask;
    a.ngroups = (int)pp.tabs.size();
    for (size_t gi = 0; gi < pp.tabs.size(); gi++) {
        const std::vector<int> &bits = pp.bits[gi];
        int nr = 0;   // runs of consecutive bits
        for (size_t j = 0; j < bits.size(); j++) {
            if (nr > 0 && bits[j] == a.rsrc[gi][nr - 1] + a.rlen[gi][nr - 1]) {
                a.rlen[gi][nr - 1]++;
                continue;
            }
            a.rsrc[gi][nr] = (uint8_t)bits[j];
            a.rdst[gi][nr] = (uint8_t)j;
            a.rlen[gi][nr] = 1;
            nr++;
        }
        a.nruns[gi] = nr;
        const auto &tab = pp.tabs[gi];
        double2 *d = nullptr;
        cuda_check(pool_malloc((void **)&d, sizeof(double2) * tab.size(), p->sv->stream), "cudaMalloc(init table)");
        cuda_check(cudaMemcpy(d, tab.data(), sizeof(double2) * tab.size(), cudaMemcpyHostToDevice), "upload init table");
        p->d_tabs.push_back(d);
        p->h2d_bytes += sizeof(double2) * tab.size();
        a.tab[gi] = d;
    }
}

// A real 1-qubit gate a·[[1, 1], [1, -1]] (Hadamard up to scale): executed as an unscaled
// butterfly (2 adds per amplitude instead of 4 FP64 ops), the factor a deferred to one global
// scale applied by the init kernel or the first tile pass (all gates are linear).
bool is_butterfly(const Gate &g, double *a) {
    if (g.kind != Kind::Dense || g.targets.size() != 1 || g.data.size() != 4) return false;
    for (auto &z : g.data)
        if (z.imag() != 0.0) return false;
    const double x = g.data[0].real();
    if (x == 0.0 || g.data[1].real() != x || g.data[2].real() != x || g.data[3].real() != -x) return false;
    if (a) *a = x;
    return true;
}

// Host-side lowering of one Tile step into register phases + op descriptors (also used by the
// host-only schedule check). Appends to blob/rops/phases; returns the first phase/op index.
// butterflies: lower Hadamard-like gates to unscaled butterflies (JIT only); prescale != 1: scale
// every amplitude by it at the start of the pass (the deferred butterfly factors).
void lower_tile_step(const Step &st, dev::TileArgs &a, std::vector<double2> &blob, std::vector<dev::RegOp> &rops,
                     std::vector<dev::RegPhase> &phases, size_t &ph0_out, size_t &opbase_out, bool butterflies,
                     double prescale) {
    auto push_data = [&](const std::vector<cplx> &d) {
        size_t off = blob.size();
        for (auto &z : d) blob.push_back(make_double2(z.real(), z.imag()));
        return off;
    };
    const size_t ph0 = phases.size();
    const size_t opbase = rops.size();
    for (size_t pi = 0; pi + 1 < st.phase_start.size(); pi++) {
        dev::RegPhase ph{};
        const std::vector<int> &Rp = st.phase_R[pi];   // physical bits, ascending
        std::vector<int> Rt;                            // tile positions
        for (int b : Rp) Rt.push_back(index_in(st.tile_bits, b));
        for (int i = 0; i < dev::kRegBits; i++) ph.R[i] = i < st.reg_bits ? Rt[i] : -1;
        int nt = 0;
        for (int tp = 0; tp < a.T; tp++)
            if (std::find(Rt.begin(), Rt.end(), tp) == Rt.end()) ph.tpos[nt++] = tp;
        ph.op0 = (int)(rops.size() - opbase);
        if (pi == 0 && prescale != 1.0) {
            dev::RegOp sc{};
            sc.kind = 3;
            sc.data_off = push_data({cplx(prescale, 0.0)});
            rops.push_back(sc);
        }
        for (size_t oi = st.phase_start[pi]; oi < st.phase_start[pi + 1]; oi++) {
            const Gate &g = st.tile_ops[oi];
            dev::RegOp r{};
            if (butterflies && is_butterfly(g, nullptr)) {
                const int rb = index_in(Rp, g.targets[0]);
                if (rb < 0) fail(SV_E_ARG, "internal: butterfly target not in registers");
                r.kind = 4;
                r.mask = 1 << rb;
                rops.push_back(r);
                continue;
            }
            auto regbit = [&](int phys_bit) { return index_in(Rp, phys_bit); };
            // route the bits of an index (table index / clock value): register slots ->
            // ridx[], thread-held tile positions and out-of-tile bits -> bit runs
            std::vector<std::pair<int, int>> tpairs, gpairs;
            auto route = [&](int b, int out) {
                const int tp = index_in(st.tile_bits, b);
                const int rg = regbit(b);
                if (rg >= 0) {
                    for (int j = 0; j < dev::kRegAmps; j++)
                        if ((j >> rg) & 1) r.ridx[j] |= 1u << out;
                } else if (tp >= 0) {
                    tpairs.push_back({tp, out});
                } else {
                    gpairs.push_back({b, out});
                }
            };
            auto to_runs = [&](std::vector<std::pair<int, int>> v, uint8_t *src, uint8_t *len,
                               uint8_t *dst, int cap) {
                std::sort(v.begin(), v.end());
                int n = 0;
                for (size_t i = 0; i < v.size(); i++) {
                    if (n > 0 && v[i].first == src[n - 1] + len[n - 1] &&
                        v[i].second == dst[n - 1] + len[n - 1]) {
                        len[n - 1]++;
                        continue;
                    }
                    if (n == cap) fail(SV_E_ARG, "internal: too many bit runs in a tile op");
                    src[n] = (uint8_t)v[i].first;
                    dst[n] = (uint8_t)v[i].second;
                    len[n] = 1;
                    n++;
                }
                return n;
            };
            if (g.kind == Kind::Dense || g.kind == Kind::Controlled) {
                r.kind = 0;
                const int k = (int)g.targets.size();
                std::vector<int> rb(k);
                for (int i = 0; i < k; i++) {
                    rb[i] = regbit(g.targets[i]);
                    if (rb[i] < 0) fail(SV_E_ARG, "internal: phase target not in registers");
                    r.mask |= 1 << rb[i];
                }
                // kernel matrix bit order = ascending register bits
                std::vector<int> order(rb);
                std::sort(order.begin(), order.end());
                std::vector<int> src(k);   // kernel bit b <- original matrix bit src[b]
                for (int bb = 0; bb < k; bb++)
                    src[bb] = (int)(std::find(rb.begin(), rb.end(), order[bb]) - rb.begin());
                const size_t D = (size_t)1 << k;
                auto orig = [&](size_t x) {
                    size_t o = 0;
                    for (int bb = 0; bb < k; bb++)
                        if ((x >> bb) & 1) o |= (size_t)1 << src[bb];
                    return o;
                };
                std::vector<cplx> Mp(D * D);
                for (size_t x = 0; x < D; x++)
                    for (size_t y = 0; y < D; y++) Mp[x * D + y] = g.data[orig(x) * D + orig(y)];
                for (size_t j = 0; j < g.controls.size(); j++) {
                    const int b = g.controls[j];
                    const int want = (int)((g.cvals >> j) & 1ull);
                    const int tp = index_in(st.tile_bits, b);
                    const int rg = regbit(b);
                    if (rg >= 0) {
                        r.rcm |= 1 << rg;
                        if (want) r.rcv |= 1 << rg;
                    } else if (tp >= 0) {
                        r.tcm |= 1u << tp;
                        if (want) r.tcv |= 1u << tp;
                    } else {
                        r.gcm |= 1ull << b;
                        if (want) r.gcv |= 1ull << b;
                    }
                }
                bool real = true;
                for (auto &z : Mp) real &= z.imag() == 0.0;
                r.is_signed = real ? 1 : 0;          // dense: real-matrix flag
                r.data_off = push_data(Mp);
            } else if (g.kind == Kind::Diagonal) {
                r.kind = 1;
                for (size_t j = 0; j < g.targets.size(); j++) route(g.targets[j], (int)j);
                // "control-like" table bits: entry == 1 whenever the bit is 0 (every CP ladder of the
                // (I)QFT). Amplitudes with such a bit 0 are left untouched: register bits skip slots,
                // thread bits / out-of-tile bits guard the op (halves the FP64 work of the ladders).
                for (size_t j = 0; j < g.targets.size(); j++) {
                    bool unit = true;
                    for (size_t idx = 0; idx < g.data.size() && unit; idx++)
                        if (!((idx >> j) & 1) && g.data[idx] != cplx(1.0, 0.0)) unit = false;
                    if (!unit) continue;
                    const int b = g.targets[j];
                    const int tp = index_in(st.tile_bits, b);
                    const int rg = regbit(b);
                    if (rg >= 0) r.rcm |= 1 << rg;
                    else if (tp >= 0) r.tcm |= 1u << tp;
                    else r.gcm |= 1ull << b;
                }
                r.rcv = r.rcm;
                r.tcv = r.tcm;
                r.gcv = r.gcm;
                r.data_off = push_data(g.data);
            } else {
                r.kind = 2;
                const int ab = regbit(g.targets[0]);
                if (ab < 0) fail(SV_E_ARG, "internal: ancilla not in registers");
                r.mask = 1 << ab;
                r.n_c = (int)g.controls.size();
                if (r.n_c > 62) fail(SV_E_ARG, "clock register too wide");
                r.is_signed = g.is_signed;
                r.dL = g.delta * std::ldexp(1.0, r.n_c - (g.is_signed ? 1 : 0));
                r.snap = g.snap;
                for (int j = 0; j < r.n_c; j++) route(g.controls[j], j);
                r.data_off = push_data({cplx(r.dL, r.snap)});
                for (auto &pr : gpairs)
                    if (pr.second >= 63) fail(SV_E_ARG, "clock register too wide for a tile");
            }
            r.ntr = to_runs(tpairs, r.t_src, r.t_len, r.t_dst, 12);
            r.ngr = to_runs(gpairs, r.g_src, r.g_len, r.g_dst, 48);
            rops.push_back(r);
        }
        ph.op1 = (int)(rops.size() - opbase);
        phases.push_back(ph);
    }
    a.nops = (int)(rops.size() - opbase);
    ph0_out = ph0;
    opbase_out = opbase;
}

sv_program *program_create(sv_state *sv, const std::vector<Gate> &ops, const std::vector<ProductFactor> *init,
                           const CompileOptions &co, uint64_t n_logical) {
    if (sv->vworld > 1) {
        std::unique_ptr<sv_program> p(new sv_program());
        p->sv = sv;
        p->n_logical = n_logical;
        p->resets = init != nullptr;
        p->phys_in = p->resets ? std::vector<int>() : sv->phys;
        try {
            for (auto *v : sv->views) {
                v->phys = sv->phys;
                p->subs.push_back(program_create(v, ops, init, co, n_logical));
            }
        } catch (...) {
            for (auto *q : p->subs) program_destroy(q);
            throw;
        }
        p->sched = p->subs[0]->sched;
        return p.release();
    }
    std::unique_ptr<sv_program> p(new sv_program());
    p->sv = sv;
    p->n_logical = n_logical;
    p->resets = init != nullptr;
    if (p->resets) {
        p->phys_in.resize(sv->n);
        std::iota(p->phys_in.begin(), p->phys_in.end(), 0);
        if ((int)co.phys_init.size() == sv->n) p->phys_in = co.phys_init;
    } else {
        p->phys_in = sv->phys;
    }
    CompileOptions c2 = co;
    if (c2.tile_qubits > 12) c2.tile_qubits = 12;
    const bool use_jit = co.jit > 0 || (co.jit == 0 && sv->nloc >= 18);
    // 8-amplitude register phases (3 register bits) only in NVRTC passes; the interpreter has 16
    c2.reg_bits = use_jit ? jit_config().reg_bits : 4;
    p->sched = compile(ops, init, sv->n, sv->nloc, p->phys_in, c2);
    prof_mark("  compile");
    const int nloc = sv->nloc;
    const uint64_t rank_base = (uint64_t)sv->rank << nloc;
    auto rank_bit = [&](int phys_bit) -> int { return (int)((rank_base >> phys_bit) & 1ull); };

    std::vector<double2> blob;
    std::vector<dev::RegOp> rops;
    std::vector<dev::RegPhase> phases;
    // deferred butterfly scale (JIT tile passes only): applied by the init or the first tile pass
    double bscale = 1.0;
    bool has_init = false;
    if (use_jit)
        for (const Step &st : p->sched.steps) {
            has_init |= st.kind == StepKind::InitProduct;
            if (st.kind != StepKind::Tile) continue;
            for (const Gate &g : st.tile_ops) {
                double x = 0.0;
                if (is_butterfly(g, &x)) bscale *= x;
            }
        }
    double pending_scale = has_init ? 1.0 : bscale;
    auto push_data = [&](const std::vector<cplx> &d) {
        size_t off = blob.size();
        for (auto &z : d) blob.push_back(make_double2(z.real(), z.imag()));
        return off;
    };
    struct Pending { size_t rec; size_t op0; size_t opbase; };
    struct GenIn {               // what a JIT pass is generated from (kept for the spill fallback)
        size_t jit;
        dev::TileArgs a;
        std::vector<dev::RegPhase> lph;
        std::vector<dev::RegOp> lops;
        bool init;
    };
    std::vector<GenIn> gen_in;
    std::vector<Pending> tiles;
    std::vector<size_t> blob_fix;     // recs whose pointer must be rebased (streaming data)

    // The product-state init fuses into the first tile pass when that pass comes right after it
    // (JIT only): the pass computes its tiles' amplitudes instead of reading them, and the init's
    // own full-state write disappears.
    const auto &steps = p->sched.steps;
    const bool fuse_init = use_jit && jit_config().init_fuse && steps.size() >= 2 &&
                           steps[0].kind == StepKind::InitProduct && steps[1].kind == StepKind::Tile;
    InitSpec init_spec;
    if (fuse_init) {
        ProductPlan pp = plan_product(sv, steps[0], bscale);
        init_spec.zero_mask = pp.zero_mask;
        for (size_t g = 0; g < pp.tabs.size(); g++) {
            init_spec.off.push_back(push_data(pp.tabs[g]));
            init_spec.bits.push_back(pp.bits[g]);
        }
        p->sched.n_passes--;
        p->sched.pass_bytes -= steps[0].bytes;                       // no separate init pass
        p->sched.pass_bytes -= 16.0 * (double)sv->local_amps();       // and the first pass reads nothing
    }
    auto gen_pass = [&](JitPass &jp, const GenIn &gi, const JitVariant &v) {
        jp.cwide.clear();
        jp.cwvals.clear();
        jp.src = gen_tile_kernel(jp.name, gi.a, gi.lph, gi.lops, &jp.smem_extra, gi.init ? &init_spec : nullptr,
                                 &jp.cwide, &blob, v);
        for (auto &c : jp.cwide)
            jp.cwvals.insert(jp.cwvals.end(), blob.begin() + c.first, blob.begin() + c.first + c.second);
    };
    // Known-zero ("lazy") qubits, JIT tile programs that start with a product init:
    // a qubit no init factor covers is |0> -- every amplitude with its bit set is 0 -- until the first
    // op that acts on it non-diagonally. If that op runs in a JIT tile pass of this program and every
    // step before it is a JIT tile pass (or the fused init), the passes before it skip the bit's
    // zero half (tiles never read or written), and the activating pass reads only the bit's zero
    // half. Exact: those amplitudes are 0 by construction (HHL: the ancilla before RECIP_RY halves
    // the first passes' traffic and FP64 work).
    std::vector<uint64_t> zin(steps.size(), 0), zout(steps.size(), 0);
    if (use_jit && fuse_init) {
        uint64_t covered = 0;
        for (auto &f : steps[0].factors)
            if (!f.diag)
                for (int q : f.qubits) covered |= 1ull << q;
        const uint64_t loc = nloc >= 64 ? ~0ull : ((1ull << nloc) - 1ull);
        uint64_t zero = loc & ~covered, eligible = zero;
        for (size_t si = 1; si < steps.size(); si++) {
            const Step &st = steps[si];
            zin[si] = zero;
            if (st.kind != StepKind::Tile) {          // non-tile step: no bit still zero here may be skipped
                eligible &= ~zero;
            }
            for (const Gate &g : st.tile_ops)
                if (g.kind == Kind::Dense || g.kind == Kind::Controlled || g.kind == Kind::RecipRY)
                    for (int q : g.targets)
                        if (q < 64) zero &= ~(1ull << q);
            if (st.kind == StepKind::Exchange) zero = 0;
            zout[si] = zero;
        }
        eligible &= ~zero;                            // never activated in this program: not skipped
        for (size_t si = 0; si < steps.size(); si++) {
            zin[si] &= eligible;
            zout[si] &= eligible;
        }
    }
    for (size_t si = 0; si < steps.size(); si++) {
        const Step &st = steps[si];
        LaunchRec rec;
        rec.kind = st.kind;
        rec.bytes = st.bytes;
        // the pass that computes the product-state init reads nothing: its HBM bytes are the write
        if (fuse_init && si == 1 && st.kind == StepKind::Tile) rec.bytes = 16.0 * (double)sv->local_amps();
        switch (st.kind) {
            case StepKind::InitZero: break;
            case StepKind::InitProduct:
                if (fuse_init) {
                    rec.skip = true;
                    rec.bytes = 0.0;
                } else if (!co.dry_run) {
                    build_product(sv, p.get(), st, rec, bscale);
                }
                break;
            case StepKind::Exchange:
                rec.xg = st.xg;
                rec.xl = st.xl;
                rec.bytes = 2.0 * 16.0 * (double)sv->local_amps() * (1.0 - std::ldexp(1.0, -(int)st.xg.size()));
                break;
            case StepKind::Dense: {
                const Gate &g = st.tile_ops[0];
                dev::DenseArgs &a = rec.dense;
                a.psi = sv->psi;
                a.k = st.k;
                std::vector<int> ins;
                for (int t = 0; t < st.k; t++) {
                    a.tpos[t] = st.tpos[t];
                    ins.push_back(st.tpos[t]);
                }
                for (size_t j = 0; j < g.controls.size(); j++) {
                    const int b = g.controls[j];
                    const int want = (int)((g.cvals >> j) & 1ull);
                    if (b >= nloc) {
                        if (rank_bit(b) != want) rec.skip = true;
                    } else {
                        ins.push_back(b);
                        if (want) a.cset |= 1ull << b;
                    }
                }
                std::sort(ins.begin(), ins.end());
                if ((int)ins.size() > dev::kMaxIns) fail(SV_E_ARG, "too many controls");
                a.nins = (int)ins.size();
                for (size_t i = 0; i < ins.size(); i++) a.ins[i] = ins[i];
                a.n_groups = 1ull << (nloc - (int)ins.size());
                rec.flops = 8.0 * std::ldexp(1.0, st.k) * std::ldexp(1.0, st.k) * (double)a.n_groups;
                a.U = reinterpret_cast<const double2 *>(push_data(g.data));
                blob_fix.push_back(p->recs.size());
                break;
            }
            case StepKind::Diagonal: {
                const Gate &g = st.tile_ops[0];
                dev::DiagArgs &a = rec.diag;
                a.psi = sv->psi;
                a.n_amps = sv->local_amps();
                a.nl = 0;
                a.gidx = 0;
                for (size_t j = 0; j < g.targets.size(); j++) {
                    const int b = g.targets[j];
                    if (b >= nloc) {
                        a.gidx |= (uint32_t)rank_bit(b) << j;
                    } else {
                        a.pos[a.nl] = b;
                        a.tbit[a.nl] = (int)j;
                        a.nl++;
                    }
                }
                a.table_len = (int)g.data.size();
                rec.flops = 6.0 * sv->local_amps();
                a.table = reinterpret_cast<const double2 *>(push_data(g.data));
                blob_fix.push_back(p->recs.size());
                break;
            }
            case StepKind::RecipRY: {
                const Gate &g = st.tile_ops[0];
                dev::RecipArgs &a = rec.recip;
                a.psi = sv->psi;
                a.n_pairs = sv->local_amps() >> 1;
                rec.flops = 6.0 * sv->local_amps();
                a.anc = g.targets[0];
                a.n_c = (int)g.controls.size();
                a.dL = g.delta * std::ldexp(1.0, a.n_c - (g.is_signed ? 1 : 0));
                a.snap = g.snap;
                a.is_signed = g.is_signed;
                a.nlc = 0;
                a.mglob = 0;
                for (int j = 0; j < a.n_c; j++) {
                    const int b = g.controls[j];
                    if (b >= nloc) {
                        a.mglob |= (uint64_t)rank_bit(b) << j;
                    } else {
                        a.lpos[a.nlc] = b;
                        a.lbit[a.nlc] = j;
                        a.nlc++;
                    }
                }
                a.contiguous = a.nlc > 0;
                for (int j = 0; j < a.nlc; j++)
                    if (a.lpos[j] != a.lpos[0] + j || a.lbit[j] != a.lbit[0] + j) a.contiguous = 0;
                if (a.contiguous) {
                    a.lo = a.lpos[0];
                    a.sh = a.lbit[0];
                    a.lmask = (a.nlc >= 64) ? ~0ull : ((1ull << a.nlc) - 1ull);
                }
                break;
            }
            case StepKind::Tile: {
                dev::TileArgs &a = rec.tile;
                a.psi = sv->psi;
                a.T = (int)st.tile_bits.size();
                a.nreg = st.reg_bits;
                for (int i = 0; i < a.T; i++) a.tbits[i] = st.tile_bits[i];
                a.nskip = 0;
                a.zload = a.zstore = 0;
                uint64_t tmask = 0;
                for (int i = 0; i < a.T; i++) tmask |= 1ull << a.tbits[i];
                for (int b = 0; b < nloc && b < 64; b++) {
                    const uint64_t m = 1ull << b;
                    if ((zin[si] & zout[si] & m) && !(tmask & m) && a.nskip < 8) a.skip[a.nskip++] = b;
                }
                for (int i = 0; i < a.T; i++) {
                    if (zin[si] >> a.tbits[i] & 1) a.zload |= 1u << i;
                    if (zout[si] >> a.tbits[i] & 1) a.zstore |= 1u << i;
                }
                a.n_tiles = 1ull << (nloc - a.T - a.nskip);
                a.nlift = 0;
                if (jit_config().xoverlap && use_jit && si + 1 < steps.size() && steps[si + 1].kind == StepKind::Exchange) {
                    // the exchange that follows takes these local bits: lift them to the top of the tile
                    // index so the pass can run slot by slot, pipelined with the transfer
                    std::vector<int> L = steps[si + 1].xl;
                    std::sort(L.begin(), L.end());
                    bool ok = L.size() <= 8;
                    for (int l : L) {
                        for (int i = 0; i < a.T; i++) ok &= a.tbits[i] != l;
                        for (int i = 0; i < a.nskip; i++) ok &= a.skip[i] != l;
                    }
                    if (ok)
                        for (int l : L) a.lift[a.nlift++] = l;
                }
                {   // HBM bytes: tiles processed x (slots read + slots written)
                    const double tiles = std::ldexp(1.0, -a.nskip);
                    const double rd = (fuse_init && si == 1) ? 0.0 : std::ldexp(1.0, -__builtin_popcount(a.zload));
                    const double wr = std::ldexp(1.0, -__builtin_popcount(a.zstore));
                    const double before = rec.bytes;      // as already counted in sched.pass_bytes
                    rec.bytes = 16.0 * (double)sv->local_amps() * tiles * (rd + wr);
                    p->sched.pass_bytes += rec.bytes - before;
                }
                a.rank_base = rank_base;
                // fused marginal: only the last step, a single-launch JIT pass over the whole (unsharded) state
                if (co.red_qubit >= 0 && co.red_qubit < sv->n && use_jit && jit_config().mred && si + 1 == steps.size() && sv->g == 0 &&
                    a.nlift == 0)
                    a.red = p->sched.phys_out[co.red_qubit];
                size_t ph0 = 0, opbase = 0;
                lower_tile_step(st, a, blob, rops, phases, ph0, opbase, use_jit, pending_scale);
                pending_scale = 1.0;
                for (size_t oi = opbase; oi < rops.size(); oi++)
                    rec.flops += regop_flops(rops[oi]) * std::ldexp((double)sv->local_amps(), -a.nskip);
                if (use_jit) {
                    GenIn gi{p->jit.size(), a, std::vector<dev::RegPhase>(phases.begin() + ph0, phases.end()),
                             std::vector<dev::RegOp>(rops.begin() + opbase, rops.end()), fuse_init && si == 1};
                    JitPass jp;           // source generated after the loop (in parallel)
                    jp.name = "hhlsv_tile";
                    jp.nthr = 1 << (a.T - a.nreg);
                    rec.jit = (int)p->jit.size();
                    p->jit.push_back(std::move(jp));
                    gen_in.push_back(std::move(gi));
                }
                a.nphase = (int)(phases.size() - ph0);
                tiles.push_back({p->recs.size(), ph0, opbase});
                break;
            }
        }
        p->recs.push_back(rec);
    }
    prof_mark("  lower");
    if (gen_in.size() == 1 || (!gen_in.empty() && sv->nloc < 24)) {     // small programs: threads cost more
        for (const GenIn &gi : gen_in) gen_pass(p->jit[gi.jit], gi, JitVariant());
    } else if (!gen_in.empty()) {       // independent per pass: shared inputs are read-only here
        std::vector<std::thread> th;
        for (const GenIn &gi : gen_in) th.emplace_back([&, pgi = &gi] { gen_pass(p->jit[pgi->jit], *pgi, JitVariant()); });
        for (auto &t : th) t.join();
    }
    prof_mark("  generate");
    // Register-spill fallback: ptxas output of every pass is checked (in parallel; the cubins are kept
    // for jit_build); a pass that spills is regenerated without constant-bank tables, then also without
    // grouped diagonal factors, keeping the variant that spills least (S33 sharded pass 3: 376 B of
    // spills, 18.6 -> 16.1 ms per rank; of the S30 passes only pass 3 spills, 8 B, at equal speed).
    // (large states only: a small program is launch- and latency-bound, spills or not)
    if (use_jit && jit_config().spillfb && !p->jit.empty() && sv->nloc >= 24) {
        std::vector<int> spill(p->jit.size(), 0);
        std::vector<size_t> unknown;          // sources not probed yet in this process
        for (size_t i = 0; i < p->jit.size(); i++)
            if (!jit_spill_cached(p->jit[i].src, &spill[i])) unknown.push_back(i);
        if (unknown.size() == 1) {
            spill[unknown[0]] = jit_spill_bytes(p->jit[unknown[0]].src);
        } else if (!unknown.empty()) {
            std::vector<std::thread> th;
            for (size_t i : unknown) th.emplace_back([&, i] { spill[i] = jit_spill_bytes(p->jit[i].src); });
            for (auto &t : th) t.join();
        }
        // the variant chosen for a default source is remembered: a repeated program regenerates only it
        static std::mutex choice_mu;
        static std::map<size_t, int> choice;        // hash of the default source -> variant (0 = default)
        const JitVariant variants[3] = {JitVariant{}, JitVariant{true, false}, JitVariant{true, true}};
        for (const GenIn &gi : gen_in) {
            int best = spill[gi.jit];
            if (best <= 0) continue;
            const size_t key = std::hash<std::string>()(p->jit[gi.jit].src);
            int known = -1;
            {
                std::lock_guard<std::mutex> lk(choice_mu);
                auto it = choice.find(key);
                if (it != choice.end()) known = it->second;
            }
            if (known >= 0) {
                if (known > 0) gen_pass(p->jit[gi.jit], gi, variants[known]);
                continue;
            }
            int pick = 0;
            for (int vi = 1; vi < 3 && best > 0; vi++) {
                JitPass alt;
                alt.name = p->jit[gi.jit].name;
                alt.nthr = p->jit[gi.jit].nthr;
                gen_pass(alt, gi, variants[vi]);
                const int s2 = jit_spill_bytes(alt.src);
                if (s2 >= 0 && s2 < best) {
                    best = s2;
                    pick = vi;
                    p->jit[gi.jit] = std::move(alt);
                }
            }
            std::lock_guard<std::mutex> lk(choice_mu);
            choice[key] = pick;
        }
    }
    prof_mark("  spill probe");
    if (co.dry_run) {       // host-only planning: compile the generated passes, log every launch
        std::string &L = *co.dry_log;
        char line[512];
        if (!co.emu_dir.empty()) {      // export for tests/jit_emulator.py (host race/bounds checking)
            auto wr = [&](const std::string &name, const void *data, size_t bytes) {
                FILE *f = fopen((co.emu_dir + "/" + name).c_str(), "wb");
                if (!f) fail(SV_E_ARG, "cannot write " + co.emu_dir + "/" + name);
                if (bytes) fwrite(data, 1, bytes, f);
                fclose(f);
            };
            wr("blob.bin", blob.data(), blob.size() * sizeof(double2));
            std::string ls;
            for (size_t i = 0; i < p->recs.size(); i++) {
                const LaunchRec &r = p->recs[i];
                if (r.kind == StepKind::Tile && r.jit >= 0) {
                    const JitPass &jp = p->jit[r.jit];
                    wr("src_" + std::to_string(i) + ".cu", jp.src.data(), jp.src.size());
                    wr("cw_" + std::to_string(i) + ".bin", jp.cwvals.data(), jp.cwvals.size() * sizeof(double2));
                    snprintf(line, sizeof line, "TILE %zu %llu %d %llu %zu %d\n", i, (unsigned long long)r.tile.n_tiles,
                             r.tile.T, (unsigned long long)r.tile.rank_base, jp.smem_extra, 1 << (r.tile.T - r.tile.nreg));
                } else if (r.skip) {
                    snprintf(line, sizeof line, "SKIP %zu %d\n", i, (int)r.kind);
                } else {
                    snprintf(line, sizeof line, "OTHER %zu %d\n", i, (int)r.kind);
                }
                ls += line;
            }
            wr("launches.txt", ls.data(), ls.size());
        }
        for (const LaunchRec &r : p->recs) {
            if (r.kind == StepKind::Tile && r.jit >= 0) {
                std::string err;
                auto cubin = jit_compile_only(p->jit[r.jit].src, err);
                if (cubin.empty()) fail(SV_E_CUDA, err);
                snprintf(line, sizeof line,
                         "JIT_PASS T=%d n_tiles=%llu skip=%d zload=%u zstore=%u bytes=%.0f flops=%.4g smem=%zu "
                         "src=%s cubin_bytes=%zu\n",
                         r.tile.T, (unsigned long long)r.tile.n_tiles, r.tile.nskip, r.tile.zload, r.tile.zstore,
                         r.bytes, r.flops, p->jit[r.jit].smem_extra, jit_source_tag(p->jit[r.jit].src).c_str(),
                         cubin.size());
            } else {
                snprintf(line, sizeof line, "LAUNCH kind=%d skip=%d bytes=%.0f\n", (int)r.kind, (int)r.skip, r.bytes);
            }
            L += line;
        }
        return p.release();
    }
    // upload blob and tile ops (stream-ordered allocations and copies, one synchronisation: the host
    // vectors live until then), then rebase pointers
    cudaStream_t us = p->sv->stream;
    if (!blob.empty()) {
        cuda_check(pool_malloc_nosync((void **)&p->d_blob, sizeof(double2) * blob.size(), us), "cudaMalloc(blob)");
        cuda_check(cudaMemcpyAsync(p->d_blob, blob.data(), sizeof(double2) * blob.size(), cudaMemcpyHostToDevice, us),
                   "upload blob");
    }
    if (!rops.empty()) {
        cuda_check(pool_malloc_nosync((void **)&p->d_ops, sizeof(dev::RegOp) * rops.size(), us), "cudaMalloc(tile ops)");
        cuda_check(cudaMemcpyAsync(p->d_ops, rops.data(), sizeof(dev::RegOp) * rops.size(), cudaMemcpyHostToDevice, us),
                   "upload tile ops");
    }
    if (!phases.empty()) {
        cuda_check(pool_malloc_nosync((void **)&p->d_phases, sizeof(dev::RegPhase) * phases.size(), us), "cudaMalloc(phases)");
        cuda_check(cudaMemcpyAsync(p->d_phases, phases.data(), sizeof(dev::RegPhase) * phases.size(),
                                   cudaMemcpyHostToDevice, us),
                   "upload phases");
    }
    cuda_check(cudaStreamSynchronize(us), "upload sync");
    p->h2d_bytes += sizeof(double2) * blob.size() + sizeof(dev::RegOp) * rops.size() +
                    sizeof(dev::RegPhase) * phases.size();
    for (size_t r : blob_fix) {
        LaunchRec &rec = p->recs[r];
        if (rec.kind == StepKind::Dense) rec.dense.U = p->d_blob + (size_t)rec.dense.U;
        if (rec.kind == StepKind::Diagonal) rec.diag.table = p->d_blob + (size_t)rec.diag.table;
    }
    prof_mark("  lower + upload");
    for (const LaunchRec &r : p->recs)
        if (r.kind == StepKind::Tile && r.jit >= 0 && r.tile.red >= 0) {
            cuda_check(pool_malloc_nosync((void **)&p->d_mred, sizeof(double) * (2 * sv_program::kMredCtas + 2), us),
                       "cudaMalloc(marginal partials)");
            p->jit[r.jit].red = p->d_mred;
        }
    if (!p->jit.empty()) jit_build(p->jit);
    prof_mark("  jit_build");
    for (auto &t : tiles) {
        p->recs[t.rec].tile.phases = p->d_phases + t.op0;
        p->recs[t.rec].tile.ops = p->d_ops + t.opbase;
        p->recs[t.rec].tile.blob = p->d_blob;
    }
    return p.release();
}

static int rec_launches(const sv_state *sv, const LaunchRec &r) {
    if (r.skip) return 0;
    if (r.kind == StepKind::Tile && r.jit >= 0 && r.tile.red >= 0) return 2;     // + the partials' sum
    if (r.kind != StepKind::Exchange) return 1;
    const XPlan x = xplan(sv, sv->rank, r.xg, r.xl);
    const uint64_t C = xchunk(x);
    const uint64_t chunks = (x.slot + C - 1) / C;
    return x.top ? 0 : (int)(2 * chunks * ((1u << x.k) - 1));   // pack + unpack kernels
}

}  // namespace hhlsv

uint64_t sv_program::launches() const {
    uint64_t n = 0;
    for (auto &r : recs) n += hhlsv::rec_launches(sv, r);
    return n;
}

namespace hhlsv {

// Pipelined pass + exchange: a JIT tile pass immediately followed by an exchange whose
// local bits are the top k local bits, none of them a tile bit or a skipped known-zero bit, splits into
// the 2^k slot ranges of the exchange -- the top k bits of the pass's tile index ARE the slot pattern,
// so tiles [p S, (p+1) S) produce exactly slot p. The slots are computed in XOR order (step d: slot
// own ^ d; the rank holding pattern own ^ d computes this rank's slot at the same step d), and slot p is sent to
// peer(p) on a communication stream while the next slot is computed: the NVLink transfer overlaps the
// pass (only slot own, kept locally, is computed first).
static bool slot_split(const sv_state *sv, const LaunchRec &tile, const LaunchRec &ex, uint64_t *per_slot) {
    if (!jit_config().xoverlap || tile.kind != StepKind::Tile || tile.jit < 0 || ex.kind != StepKind::Exchange ||
        tile.skip)
        return false;
    const XPlan x = xplan(sv, sv->rank, ex.xg, ex.xl);
    if (tile.tile.nlift != x.k) return false;
    for (int i = 0; i < x.k; i++)
        if (tile.tile.lift[i] != x.Ls[i]) return false;
    const uint64_t n = tile.tile.n_tiles;
    if ((n >> x.k) << x.k != n || (n >> x.k) == 0) return false;
    *per_slot = n >> x.k;
    return true;
}

// Send slot p to peer(p) and receive peer(p)'s slot into it, chunked, on stream cs (contiguous slots
// straight from the state, others through the pack / unpack kernels).
static void exchange_slot(sv_state *sv, const XPlan &x, uint32_t p, cudaStream_t cs) {
    const uint64_t C = xchunk(x);
    ensure_xbuf(sv, C);
    const int peer = xpeer(sv, x, sv->rank, p);
    for (uint64_t off = 0; off < x.slot; off += C) {
        const uint64_t cnt = std::min(C, x.slot - off);
        const double *sb = (const double *)(sv->psi + (uint64_t)p * x.slot + off);
        if (!x.top) {
            cuda_check(dev::launch_pack_multi(sv->psi, sv->d_xsend, x.Ls.data(), x.k, p, off, cnt, cs), "slot pack");
            sb = (const double *)sv->d_xsend;
        }
        double *rb = (double *)sv->d_xrecv;
        nccl_check(nccl_alltoall_pairs(sv->comm, &sb, &rb, &peer, 1, 2 * cnt, cs), "exchange slot");
        if (x.top)
            cuda_check(cudaMemcpyAsync(sv->psi + (uint64_t)p * x.slot + off, sv->d_xrecv, sizeof(double2) * cnt,
                                       cudaMemcpyDeviceToDevice, cs),
                       "exchange slot copy");
        else
            cuda_check(dev::launch_unpack_multi(sv->psi, sv->d_xrecv, x.Ls.data(), x.k, p, off, cnt, cs), "slot unpack");
    }
}

// One JIT tile pass over all its tiles; a pass with the fused marginal also sums its CTA partials.
static void launch_jit_rec(sv_state *sv, sv_program *p, const LaunchRec &r) {
    const JitPass &jp = p->jit[r.jit];
    cuda_check(jit_launch(jp, r.tile.psi, r.tile.blob, r.tile.n_tiles, r.tile.rank_base, r.tile.T, sv->stream),
               "tile (jit)");
    if (jp.red) {
        const uint64_t grid = jit_grid(jp, r.tile.n_tiles);
        if (grid > (uint64_t)sv_program::kMredCtas) fail(SV_E_CUDA, "fused marginal: launch grid too large");
        cuda_check(dev::launch_pair_sum(jp.red, (int)grid, jp.red + 2 * sv_program::kMredCtas, sv->stream),
                   "marginal partial sum");
    }
}

static void launch_rec(sv_state *sv, sv_program *p, const LaunchRec &r) {
    if (r.skip) return;
    switch (r.kind) {
        case StepKind::InitZero: cuda_check(dev::launch_zero_init(sv->psi, sv->local_amps(), sv->rank == 0, sv->stream), "init"); break;
        case StepKind::InitProduct: cuda_check(dev::launch_product(r.prod, sv->stream), "product init"); break;
        case StepKind::Dense: cuda_check(dev::launch_dense(r.dense, sv->stream), "dense"); break;
        case StepKind::Diagonal: cuda_check(dev::launch_diag(r.diag, sv->stream), "diagonal"); break;
        case StepKind::RecipRY: cuda_check(dev::launch_recip(r.recip, sv->stream), "recip_ry"); break;
        case StepKind::Tile:
            if (r.jit >= 0)
                launch_jit_rec(sv, p, r);
            else
                cuda_check(dev::launch_tile(r.tile, sv->stream), "tile");
            break;
        case StepKind::Exchange: break;
    }
}

void program_run(sv_state *sv, sv_program *p) {
    if (p->sv != sv) fail(SV_E_ARG, "program belongs to another state");
    if (!p->resets && sv->phys != p->phys_in) fail(SV_E_ARG, "qubit map changed since the program was created");
    if (!p->subs.empty()) {             // virtual sharding: step-interleaved over the shards
        const size_t ns = p->subs[0]->recs.size();
        sv_program *t0 = p->subs[0];     // timing: one event pair per step, spanning every shard's launches
        if (p->timing && t0->ev.size() != 2 * ns) {
            for (auto e : t0->ev) cudaEventDestroy(e);
            t0->ev.assign(2 * ns, nullptr);
            for (auto &e : t0->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        }
        for (size_t i = 0; i < ns; i++) {
            if (p->timing) cuda_check(cudaEventRecord(t0->ev[2 * i], sv->stream), "event");
            struct EndEv {
                sv_program *p, *t0;
                sv_state *sv;
                size_t i;
                ~EndEv() {
                    if (p->timing) cudaEventRecord(t0->ev[2 * i + 1], sv->stream);
                }
            } end_ev{p, t0, sv, i};
            if (p->subs[0]->recs[i].kind == StepKind::Exchange) {
                virtual_exchange(sv, p->subs[0]->recs[i].xg, p->subs[0]->recs[i].xl);
                continue;
            }
            uint64_t per = 0;
            if (i + 1 < ns && slot_split(sv->views[0], p->subs[0]->recs[i], p->subs[0]->recs[i + 1], &per)) {
                // the slot-range launches of the pipelined path (same kernels, same ranges)
                const XPlan x0 = xplan(sv->views[0], 0, p->subs[0]->recs[i + 1].xg, p->subs[0]->recs[i + 1].xl);
                for (size_t r = 0; r < p->subs.size(); r++) {
                    const LaunchRec &tr = p->subs[r]->recs[i];
                    const uint32_t own = xplan(sv->views[r], (int)r, p->subs[r]->recs[i + 1].xg,
                                               p->subs[r]->recs[i + 1].xl).own;
                    for (uint32_t d = 0; d < (1u << x0.k); d++) {
                        const uint64_t slot = own ^ d;
                        cuda_check(jit_launch(p->subs[r]->jit[tr.jit], tr.tile.psi, tr.tile.blob, (slot + 1) * per,
                                              tr.tile.rank_base, tr.tile.T, sv->stream, slot * per),
                                   "tile (jit, slot range)");
                    }
                }
                continue;
            }
            for (size_t r = 0; r < p->subs.size(); r++) launch_rec(sv->views[r], p->subs[r], p->subs[r]->recs[i]);
        }
        sv->phys = p->sched.phys_out;
        for (auto *v : sv->views) v->phys = sv->phys;
        return;
    }
    // CUDA graph for small single-rank programs (launch-bound: Table 1's 13-16 qubit circuits run a few
    // passes of tens of microseconds): the launches of the second run are captured on a private stream
    // and replayed from then on, ordered after / before the state's stream by events
    bool graphable = sv->world == 1 && !p->timing && sv->local_amps() <= (1ull << 20) && jit_config().graphs;
    for (const LaunchRec &r : p->recs) graphable &= r.kind != StepKind::Exchange;
    if (graphable && ++p->runs >= 2) {
        if (!p->gstream) {
            cuda_check(cudaStreamCreateWithFlags(&p->gstream, cudaStreamNonBlocking), "graph stream");
            cuda_check(cudaEventCreateWithFlags(&p->gev_a, cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&p->gev_b, cudaEventDisableTiming), "event");
        }
        cuda_check(cudaEventRecord(p->gev_a, sv->stream), "event");
        cuda_check(cudaStreamWaitEvent(p->gstream, p->gev_a, 0), "wait");
        if (!p->graph_exec) {
            cudaStream_t user = sv->stream;
            sv->stream = p->gstream;                         // launch_rec enqueues on sv->stream
            cuda_check(cudaStreamBeginCapture(p->gstream, cudaStreamCaptureModeThreadLocal), "begin capture");
            for (const LaunchRec &r : p->recs) launch_rec(sv, p, r);
            const cudaError_t ce = cudaStreamEndCapture(p->gstream, &p->graph);
            sv->stream = user;
            cuda_check(ce, "end capture");
            cuda_check(cudaGraphInstantiate(&p->graph_exec, p->graph, 0), "graph instantiate");
        }
        cuda_check(cudaGraphLaunch(p->graph_exec, p->gstream), "graph launch");
        cuda_check(cudaEventRecord(p->gev_b, p->gstream), "event");
        cuda_check(cudaStreamWaitEvent(sv->stream, p->gev_b, 0), "wait");
        sv->phys = p->sched.phys_out;
        return;
    }
    if (p->timing && p->ev.size() != 2 * p->recs.size()) {
        for (auto e : p->ev) cudaEventDestroy(e);
        p->ev.assign(2 * p->recs.size(), nullptr);
        for (auto &e : p->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    }
    for (size_t ri = 0; ri < p->recs.size(); ri++) {
        const LaunchRec &r = p->recs[ri];
        if (p->timing) cuda_check(cudaEventRecord(p->ev[2 * ri], sv->stream), "event");
        uint64_t per = 0;
        if (sv->world > 1 && ri + 1 < p->recs.size() && slot_split(sv, r, p->recs[ri + 1], &per)) {
            const LaunchRec &ex = p->recs[ri + 1];
            const XPlan x = xplan(sv, sv->rank, ex.xg, ex.xl);
            if (!sv->comm_stream) cuda_check(cudaStreamCreateWithFlags(&sv->comm_stream, cudaStreamNonBlocking), "comm stream");
            if (!sv->ev_a) {
                cuda_check(cudaEventCreateWithFlags(&sv->ev_a, cudaEventDisableTiming), "event");
                cuda_check(cudaEventCreateWithFlags(&sv->ev_b, cudaEventDisableTiming), "event");
            }
            nvtxRangePushA("hhlsv tile_pass+exchange (pipelined)");
            for (uint32_t d = 0; d < (1u << x.k); d++) {
                const uint32_t slot = x.own ^ d;
                cuda_check(jit_launch(p->jit[r.jit], r.tile.psi, r.tile.blob, (slot + 1) * per, r.tile.rank_base, r.tile.T,
                                      sv->stream, (uint64_t)slot * per),
                           "tile (jit, slot range)");
                if (d == 0) continue;                    // own slot: stays here
                cuda_check(cudaEventRecord(sv->ev_a, sv->stream), "event");
                cuda_check(cudaStreamWaitEvent(sv->comm_stream, sv->ev_a, 0), "wait");
                exchange_slot(sv, x, slot, sv->comm_stream);
            }
            if (p->timing) {
                cuda_check(cudaEventRecord(p->ev[2 * ri + 1], sv->stream), "event");
                cuda_check(cudaEventRecord(p->ev[2 * ri + 2], sv->stream), "event");
            }
            cuda_check(cudaEventRecord(sv->ev_b, sv->comm_stream), "event");
            cuda_check(cudaStreamWaitEvent(sv->stream, sv->ev_b, 0), "wait");
            nvtxRangePop();
            ri++;                                        // the exchange step is done
            if (p->timing) cuda_check(cudaEventRecord(p->ev[2 * ri + 1], sv->stream), "event");
            continue;
        }
        if (r.skip) {
            if (p->timing) cuda_check(cudaEventRecord(p->ev[2 * ri + 1], sv->stream), "event");
            continue;
        }
        // NVTX range per step (SURVEY §5 tracing): one per tile pass / streaming op / exchange, named by
        // kind and step index; a no-op unless a tool (nsys, ncu --nvtx) is attached
        static const char *knames[] = {"init_zero", "init_product", "dense", "diagonal", "recip_ry", "tile_pass",
                                       "exchange"};
        char rname[64];
        snprintf(rname, sizeof rname, "hhlsv %s #%zu", knames[(int)r.kind], ri);
        nvtxRangePushA(rname);
        switch (r.kind) {
            case StepKind::InitZero: cuda_check(dev::launch_zero_init(sv->psi, sv->local_amps(), sv->rank == 0, sv->stream), "init"); break;
            case StepKind::InitProduct: cuda_check(dev::launch_product(r.prod, sv->stream), "product init"); break;
            case StepKind::Dense: cuda_check(dev::launch_dense(r.dense, sv->stream), "dense"); break;
            case StepKind::Diagonal: cuda_check(dev::launch_diag(r.diag, sv->stream), "diagonal"); break;
            case StepKind::RecipRY: cuda_check(dev::launch_recip(r.recip, sv->stream), "recip_ry"); break;
            case StepKind::Tile:
                if (r.jit >= 0)
                    launch_jit_rec(sv, p, r);
                else
                    cuda_check(dev::launch_tile(r.tile, sv->stream), "tile");
                break;
            case StepKind::Exchange: exchange(sv, r.xg, r.xl); break;
        }
        nvtxRangePop();
        if (p->timing) cuda_check(cudaEventRecord(p->ev[2 * ri + 1], sv->stream), "event");
    }
    sv->phys = p->sched.phys_out;
}

void program_timings(sv_program *p, float *ms, int *kind, double *bytes, double *flops, int *launches, size_t cap,
                     size_t *n_out) {
    if (!p->subs.empty()) {      // virtual shards: per step over all shards (bytes / flops / launches summed)
        sv_program *t0 = p->subs[0];
        if (!p->timing || t0->ev.size() != 2 * t0->recs.size()) fail(SV_E_ARG, "timing not enabled or program not run");
        cuda_check(cudaStreamSynchronize(p->sv->stream), "timings sync");
        const size_t n = std::min(cap, t0->recs.size());
        for (size_t i = 0; i < n; i++) {
            float t = 0.0f;
            cuda_check(cudaEventElapsedTime(&t, t0->ev[2 * i], t0->ev[2 * i + 1]), "elapsed");
            if (ms) ms[i] = t;
            if (kind) kind[i] = (int)t0->recs[i].kind;
            double by = 0, fl = 0;
            int la = 0;
            for (size_t r = 0; r < p->subs.size(); r++) {
                by += p->subs[r]->recs[i].bytes;
                fl += p->subs[r]->recs[i].flops;
                la += rec_launches(p->subs[r]->sv, p->subs[r]->recs[i]);
            }
            if (bytes) bytes[i] = by;
            if (flops) flops[i] = fl;
            if (launches) launches[i] = la;
        }
        if (n_out) *n_out = t0->recs.size();
        return;
    }
    if (!p->timing || p->ev.size() != 2 * p->recs.size()) fail(SV_E_ARG, "timing not enabled or program not run");
    cuda_check(cudaStreamSynchronize(p->sv->stream), "timings sync");
    const size_t n = std::min(cap, p->recs.size());
    for (size_t i = 0; i < n; i++) {
        float t = 0.0f;
        cuda_check(cudaEventElapsedTime(&t, p->ev[2 * i], p->ev[2 * i + 1]), "elapsed");
        if (ms) ms[i] = t;
        if (kind) kind[i] = (int)p->recs[i].kind;
        if (bytes) bytes[i] = p->recs[i].bytes;
        if (flops) flops[i] = p->recs[i].flops;
        if (launches) launches[i] = rec_launches(p->sv, p->recs[i]);
    }
    if (n_out) *n_out = p->recs.size();
}

void program_destroy(sv_program *p) {
    if (!p) return;
    if (p->sv) cudaStreamSynchronize(p->sv->stream);
    for (auto *q : p->subs) program_destroy(q);
    pool_free(p->d_blob, p->sv ? p->sv->stream : nullptr);
    pool_free(p->d_ops, p->sv ? p->sv->stream : nullptr);
    pool_free(p->d_phases, p->sv ? p->sv->stream : nullptr);
    for (auto *d : p->d_tabs) pool_free(d, p->sv ? p->sv->stream : nullptr);
    pool_free(p->d_mred, p->sv ? p->sv->stream : nullptr);
    for (auto e : p->ev) cudaEventDestroy(e);
    if (p->graph_exec) cudaGraphExecDestroy(p->graph_exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    if (p->gstream) cudaStreamDestroy(p->gstream);
    if (p->gev_a) cudaEventDestroy(p->gev_a);
    if (p->gev_b) cudaEventDestroy(p->gev_b);
    delete p;
}

// ---------------------------------------------------------------- readout ----
static void allreduce_if_sharded(sv_state *sv, double *dbuf, size_t count) {
    if (sv->world > 1) nccl_check(nccl_allreduce_sum(sv->comm, dbuf, count, sv->stream), "allreduce");
}

// Stream synchronisation of a readout. Sharded states: poll with NCCL failure detection (asynchronous
// communicator errors, a 300 s timeout for a lost peer) instead of blocking forever.
static void sync_readout(sv_state *sv, const char *what) {
    if (sv->world > 1) nccl_check(nccl_wait(sv->comm, sv->stream, 300.0), what);
    else cuda_check(cudaStreamSynchronize(sv->stream), what);
}

double state_norm2(sv_state *sv) {
    if (sv->vworld > 1) {
        double t = 0.0;
        for (auto *v : sv->views) t += state_norm2(v);
        return t;
    }
    cuda_check(dev::launch_norm2(sv->psi, sv->local_amps(), sv->d_red, sv->d_scalar, sv->stream), "norm2");
    allreduce_if_sharded(sv, sv->d_scalar, 1);
    double h = 0.0;
    cuda_check(cudaMemcpyAsync(&h, sv->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, sv->stream), "norm2 d2h");
    sync_readout(sv, "norm2 sync");
    return h;
}

void state_probabilities(sv_state *sv, const int *qubits, int nq, double *out) {
    if (nq < 0 || nq > 26 || (nq > 0 && !qubits) || !out) fail(SV_E_ARG, "probabilities: bad qubit list");
    if (sv->vworld > 1) {
        const size_t nout = (size_t)1 << nq;
        std::vector<double> part(nout);
        std::fill(out, out + nout, 0.0);
        for (auto *v : sv->views) {
            v->phys = sv->phys;
            state_probabilities(v, qubits, nq, part.data());
            for (size_t i = 0; i < nout; i++) out[i] += part[i];
        }
        return;
    }
    std::vector<int> q(qubits, qubits + nq);
    for (int i = 0; i < nq; i++) {
        if (q[i] < 0 || q[i] >= sv->n) fail(SV_E_ARG, "probabilities: qubit out of range");
        for (int j = 0; j < i; j++)
            if (q[i] == q[j]) fail(SV_E_ARG, "probabilities: duplicated qubit");
    }
    std::vector<int> S, jpos;
    uint64_t gv = 0;
    for (int j = 0; j < nq; j++) {
        const int b = sv->phys[q[j]];
        if (b < sv->nloc) {
            S.push_back(b);
            jpos.push_back(j);
        } else if ((sv->rank >> (b - sv->nloc)) & 1) {
            gv |= 1ull << j;
        }
    }
    const int ql = (int)S.size();
    const size_t C = (size_t)dev::marginal_chunks(sv->nloc, ql);
    ensure_red(sv, ((size_t)1 << ql) * C + ((size_t)1 << ql));
    double *ws = sv->d_red;
    double *dout = sv->d_red + ((size_t)1 << ql) * C;
    cuda_check(dev::launch_marginal(sv->psi, sv->nloc, S.data(), ql, ws, dout, sv->stream), "marginal");
    std::vector<double> loc((size_t)1 << ql);
    cuda_check(cudaMemcpyAsync(loc.data(), dout, sizeof(double) * loc.size(), cudaMemcpyDeviceToHost, sv->stream),
               "marginal d2h");
    cuda_check(cudaStreamSynchronize(sv->stream), "marginal sync");
    const size_t nout = (size_t)1 << nq;
    std::fill(out, out + nout, 0.0);
    for (size_t v = 0; v < loc.size(); v++) {
        uint64_t o = gv;
        for (int i = 0; i < ql; i++)
            if ((v >> i) & 1) o |= 1ull << jpos[i];
        out[o] = loc[v];
    }
    if (sv->world > 1) {
        ensure_red(sv, nout);
        cuda_check(cudaMemcpyAsync(sv->d_red, out, sizeof(double) * nout, cudaMemcpyHostToDevice, sv->stream), "h2d");
        allreduce_if_sharded(sv, sv->d_red, nout);
        cuda_check(cudaMemcpyAsync(out, sv->d_red, sizeof(double) * nout, cudaMemcpyDeviceToHost, sv->stream), "d2h");
        sync_readout(sv, "probabilities sync");
    }
}

static void fill_phys(const sv_state *sv, int *dst) {
    for (int q = 0; q < sv->n; q++) dst[q] = sv->phys[q];
}

void state_read(sv_state *sv, uint64_t first, uint64_t count, double *out) {
    const uint64_t N = 1ull << sv->n;
    if (first > N || count > N - first) fail(SV_E_RANGE, "read: range outside the state");
    if (count && !out) fail(SV_E_ARG, "read: null output");
    if (sv->vworld > 1) {
        std::vector<double> part(2 * count);
        std::fill(out, out + 2 * count, 0.0);
        for (auto *v : sv->views) {
            v->phys = sv->phys;
            state_read(v, first, count, part.data());
            for (uint64_t i = 0; i < 2 * count; i++) out[i] += part[i];
        }
        return;
    }
    const uint64_t chunk = 1ull << 22;
    ensure_io(sv, std::min(count, chunk));
    for (uint64_t off = 0; off < count; off += chunk) {
        const uint64_t c = std::min(chunk, count - off);
        dev::GatherArgs a{};
        a.psi = sv->psi;
        a.out = sv->d_io;
        a.count = c;
        a.first = first + off;
        a.n = sv->n;
        a.nloc = sv->nloc;
        a.rank = (uint64_t)sv->rank;
        fill_phys(sv, a.phys);
        cuda_check(dev::launch_gather(a, sv->stream), "gather");
        allreduce_if_sharded(sv, (double *)sv->d_io, 2 * c);
        cuda_check(cudaMemcpyAsync(out + 2 * off, sv->d_io, sizeof(double2) * c, cudaMemcpyDeviceToHost, sv->stream),
                   "read d2h");
    }
    sync_readout(sv, "read sync");
}

void state_write(sv_state *sv, uint64_t first, uint64_t count, const double *in) {
    const uint64_t N = 1ull << sv->n;
    if (first > N || count > N - first) fail(SV_E_RANGE, "write: range outside the state");
    if (count && !in) fail(SV_E_ARG, "write: null input");
    if (sv->vworld > 1) {
        for (auto *v : sv->views) {
            v->phys = sv->phys;
            state_write(v, first, count, in);
        }
        return;
    }
    const uint64_t chunk = 1ull << 22;
    ensure_io(sv, std::min(count, chunk));
    for (uint64_t off = 0; off < count; off += chunk) {
        const uint64_t c = std::min(chunk, count - off);
        cuda_check(cudaMemcpyAsync(sv->d_io, in + 2 * off, sizeof(double2) * c, cudaMemcpyHostToDevice, sv->stream),
                   "write h2d");
        dev::ScatterArgs a{};
        a.psi = sv->psi;
        a.in = sv->d_io;
        a.count = c;
        a.first = first + off;
        a.n = sv->n;
        a.nloc = sv->nloc;
        a.rank = (uint64_t)sv->rank;
        fill_phys(sv, a.phys);
        cuda_check(dev::launch_scatter(a, sv->stream), "scatter");
    }
    cuda_check(cudaStreamSynchronize(sv->stream), "write sync");
}

void state_sample(sv_state *sv, uint64_t shots, uint64_t seed, uint64_t *out) {
    if (sv->world > 1 || sv->vworld > 1) fail(SV_E_ARG, "sample: single-rank states only");
    if (shots && !out) fail(SV_E_ARG, "sample: null output");
    std::unique_ptr<dev::SampleArgs> a(new dev::SampleArgs());
    a->psi = sv->psi;
    a->n = sv->n;
    a->lb1 = std::min(sv->n, dev::kSampleLB1);
    a->nblk = 1ull << (sv->n - a->lb1);
    a->lb2 = std::min(sv->n - a->lb1, dev::kSampleLB2);
    a->nsup = a->nblk >> a->lb2;
    fill_phys(sv, a->phys);
    for (uint64_t i = 0; i < (1ull << a->lb1); i++) {
        uint64_t P = 0;
        for (int q = 0; q < a->lb1; q++)
            if ((i >> q) & 1ull) P |= 1ull << a->phys[q];
        a->lo[i] = P;
    }
    a->shots = shots;
    a->seed = seed;
    cuda_check(pool_malloc((void **)&a->S, sizeof(double) * a->nblk, sv->stream), "alloc(sample S)");
    cuda_check(pool_malloc((void **)&a->cum, sizeof(double) * a->nsup, sv->stream), "alloc(sample cum)");
    cuda_check(pool_malloc((void **)&a->out, sizeof(uint64_t) * std::max<uint64_t>(1, shots), sv->stream),
               "alloc(sample out)");
    struct Free {
        sv_state *sv;
        dev::SampleArgs *a;
        ~Free() {
            pool_free(a->S, sv->stream);
            pool_free(a->cum, sv->stream);
            pool_free(a->out, sv->stream);
        }
    } fr{sv, a.get()};
    cuda_check(dev::launch_sample_sums(*a, sv->stream), "sample sums");
    double total = 0.0;
    cuda_check(cudaMemcpyAsync(&total, a->cum + a->nsup - 1, sizeof(double), cudaMemcpyDeviceToHost, sv->stream),
               "sample total");
    cuda_check(cudaStreamSynchronize(sv->stream), "sample sync");
    if (!(total > 0.0)) fail(SV_E_ZEROPROB, "sample: zero state");
    cuda_check(dev::launch_sample_draw(*a, sv->stream), "sample draw");
    if (shots)
        cuda_check(cudaMemcpyAsync(out, a->out, sizeof(uint64_t) * shots, cudaMemcpyDeviceToHost, sv->stream),
                   "sample out");
    cuda_check(cudaStreamSynchronize(sv->stream), "sample sync");
}

void state_postselect(sv_state *sv, const int *fq, const int *fv, int nfixed, double *amps, uint64_t *idx,
                      uint64_t n_out, double *prob) {
    if (nfixed < 0 || (nfixed > 0 && (!fq || !fv)) || !amps) fail(SV_E_ARG, "postselect: bad arguments");
    uint64_t fixed = 0, fmask = 0;
    for (int i = 0; i < nfixed; i++) {
        if (fq[i] < 0 || fq[i] >= sv->n || (fmask >> fq[i]) & 1ull) fail(SV_E_ARG, "postselect: bad qubit");
        if (fv[i] != 0 && fv[i] != 1) fail(SV_E_ARG, "postselect: values must be 0/1");
        fmask |= 1ull << fq[i];
        if (fv[i]) fixed |= 1ull << fq[i];
    }
    if (sv->vworld > 1) {
        std::vector<double> part(2 * n_out);
        std::fill(amps, amps + 2 * n_out, 0.0);
        for (auto *v : sv->views) {
            v->phys = sv->phys;
            state_postselect(v, fq, fv, nfixed, part.data(), idx, n_out, nullptr);
            for (uint64_t i = 0; i < 2 * n_out; i++) amps[i] += part[i];
        }
        if (prob) {
            double s = 0.0;
            for (uint64_t e = 0; e < 2 * n_out; e++) s += amps[e] * amps[e];
            *prob = s;
        }
        return;
    }
    dev::GatherArgs a{};
    int nfree = 0;
    for (int q = 0; q < sv->n; q++)
        if (!((fmask >> q) & 1ull)) a.free_q[nfree++] = q;
    if (nfree > 26 || n_out != (1ull << nfree)) fail(SV_E_ARG, "postselect: n_out must be 2^(n - n_fixed) <= 2^26");
    ensure_io(sv, n_out);
    a.psi = sv->psi;
    a.out = sv->d_io;
    a.count = n_out;
    a.first = 0;
    a.n = sv->n;
    a.nloc = sv->nloc;
    a.rank = (uint64_t)sv->rank;
    fill_phys(sv, a.phys);
    a.nfree = nfree == 0 ? -1 : nfree;   // -1: only the fixed index
    if (nfree == 0) {
        a.nfree = 1;                     // deposit of 0 -> fixed (free_q[0] unused for x=0)
        a.free_q[0] = 0;
    }
    a.fixed = fixed;
    cuda_check(dev::launch_gather(a, sv->stream), "postselect gather");
    allreduce_if_sharded(sv, (double *)sv->d_io, 2 * n_out);
    cuda_check(cudaMemcpyAsync(amps, sv->d_io, sizeof(double2) * n_out, cudaMemcpyDeviceToHost, sv->stream),
               "postselect d2h");
    sync_readout(sv, "postselect sync");
    if (idx)
        for (uint64_t e = 0; e < n_out; e++) {
            uint64_t L = fixed;
            for (int i = 0; i < nfree; i++)
                if ((e >> i) & 1ull) L |= 1ull << a.free_q[i];
            idx[e] = L;
        }
    if (prob) {
        double s = 0.0;
        for (uint64_t e = 0; e < 2 * n_out; e++) s += amps[e] * amps[e];
        *prob = s;
    }
}

}  // namespace hhlsv
