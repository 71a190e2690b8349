// sm_100a kernels of the HHL state-vector hot path.
//
// Every kernel streams the interleaved complex128 state in HBM with 16-byte (double2)
// accesses, 64-bit index arithmetic, grid-stride loops sized in multiples of the 148 SMs,
// and fp64 FMA arithmetic (the paper's precision is fp64 complex; R16).
// Reductions are fixed-order trees (warp shuffle -> block -> grid), never fp64 atomics,
// so two runs are bit-identical.
#include <cstdio>

#include "jit.h"
#include "kernels.cuh"

namespace hhlsv {
namespace dev {

constexpr int kThreads = 256;
constexpr int kSMs = 148;

__device__ __forceinline__ uint64_t insz(uint64_t x, int p) {
    const uint64_t lo = x & ((1ull << p) - 1ull);
    return ((x >> p) << (p + 1)) | lo;
}

__device__ __forceinline__ void cfma(double2 &acc, const double2 a, const double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

__device__ __forceinline__ double2 cmul(const double2 a, const double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// Reciprocal rotation sine, SURVEY §8(a) a7 / DESIGN.md R6 (identical IEEE operations to the
// oracle's definition so that the snapping/clipping decisions agree bit for bit).
__device__ __forceinline__ double recip_s(uint64_t m, int n_c, double dL, int is_signed, double snap) {
    if (m == 0) return 0.0;
    double sign = 1.0;
    uint64_t mp = m;
    if (is_signed && m >= (1ull << (n_c - 1))) {
        mp = (1ull << n_c) - m;
        sign = -1.0;
    }
    const double r = __ddiv_rn(dL, (double)mp);
    const double s = fabs(r - 1.0) <= snap ? 1.0 : (r < 1.0 ? r : 0.0);
    return sign * s;
}

static int grid_for(uint64_t work, int per_block) {
    uint64_t b = (work + per_block - 1) / per_block;
    const uint64_t cap = (uint64_t)kSMs * 8;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// ============================================================ a4/a5 dense ====
// One thread per group of 2^K amplitudes (G groups per thread for small K to keep
// >= 8 independent 16-byte loads in flight). The matrix sits in shared memory and is
// read as a warp-wide broadcast.
template <int K, int G>
__global__ void __launch_bounds__(kThreads) k_dense(const DenseArgs a) {
    constexpr int D = 1 << K;
    __shared__ double2 sU[D * D];
    __shared__ uint64_t soff[D];
    for (int i = threadIdx.x; i < D * D; i += blockDim.x) sU[i] = a.U[i];
    if (threadIdx.x < D) {
        uint64_t o = 0;
        for (int i = 0; i < K; i++)
            if ((threadIdx.x >> i) & 1) o |= 1ull << a.tpos[i];
        soff[threadIdx.x] = o;
    }
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * G;
    for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x * G + threadIdx.x; g0 < a.n_groups; g0 += stride) {
        uint64_t base[G];
        double2 v[G][D];
#pragma unroll
        for (int gg = 0; gg < G; gg++) {
            uint64_t g = g0 + (uint64_t)gg * blockDim.x;
            if (g >= a.n_groups) g = g0;          // duplicate work on the tail, stores are idempotent
            uint64_t b = g;
            for (int i = 0; i < a.nins; i++) b = insz(b, a.ins[i]);
            base[gg] = b | a.cset;
#pragma unroll
            for (int c = 0; c < D; c++) v[gg][c] = a.psi[base[gg] | soff[c]];
        }
#pragma unroll
        for (int gg = 0; gg < G; gg++) {
            // rows in blocks of RB independent accumulators (FMA latency hidden by 2 RB chains); the
            // block loop is not unrolled for K >= 3 so the compiler cannot hoist the whole matrix out of
            // the grid-stride loop into registers
            constexpr int RB = D < 4 ? D : 4;
#pragma unroll(K >= 3 ? 1 : D / RB)
            for (int r0 = 0; r0 < D; r0 += RB) {
                double2 acc[RB];
#pragma unroll
                for (int rr = 0; rr < RB; rr++) acc[rr] = make_double2(0.0, 0.0);
#pragma unroll
                for (int c = 0; c < D; c++)
#pragma unroll
                    for (int rr = 0; rr < RB; rr++) cfma(acc[rr], sU[(r0 + rr) * D + c], v[gg][c]);
#pragma unroll
                for (int rr = 0; rr < RB; rr++) a.psi[base[gg] | soff[r0 + rr]] = acc[rr];
            }
        }
    }
}

// k = 5 on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): the only dense contraction of the path
// (256 flop per amplitude, FP64-bound). The 32 x 32 complex matrix is the real 64 x 64
// block matrix M = [[Ur, -Ui], [Ui, Ur]] in shared memory (rows padded to 68 doubles: 2 wavefronts
// per A-fragment load). A warp takes 8 groups at a time: lane (n = lane / 4, kk = lane % 4) holds, as
// its 16 B fragments, re / im of amplitudes kk, kk + 4, ..., kk + 28 of group n; 8 row tiles x 16
// k-steps = 128 DMMAs give Y = M X (64 x 8), and the lane owning output rows e and e + 32 (re, im of
// amplitude e) writes them back for its two groups. Each group is read completely into registers
// before any write (in place, groups disjoint across warps).
template <int K>
__global__ void __launch_bounds__(kThreads) k_dense_dmma(const DenseArgs a, uint64_t n_batches) {
    constexpr int D = 1 << K;          // complex dimension
    constexpr int R = 2 * D;           // real dimension of M
    constexpr int P = R + 4;           // padded row (doubles)
    __shared__ double sM[R * P];
    __shared__ uint64_t soff[D];
    for (int i = threadIdx.x; i < D * D; i += blockDim.x) {
        const int r = i / D, c = i % D;
        const double2 u = a.U[i];
        sM[r * P + c] = u.x;
        sM[r * P + D + c] = -u.y;
        sM[(D + r) * P + c] = u.y;
        sM[(D + r) * P + D + c] = u.x;
    }
    if (threadIdx.x < D) {
        uint64_t o = 0;
        for (int i = 0; i < K; i++)
            if ((threadIdx.x >> i) & 1) o |= 1ull << a.tpos[i];
        soff[threadIdx.x] = o;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, n = lane >> 2, kk = lane & 3;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t bt = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); bt < n_batches; bt += warps) {
        uint64_t b = bt * 8 + n;                   // this lane's group
        for (int i = 0; i < a.nins; i++) b = insz(b, a.ins[i]);
        b |= a.cset;
        double xr[D / 4], xi[D / 4];               // B fragments: x[4 ks + kk], re for ks < D/4, im after
#pragma unroll
        for (int q = 0; q < D / 4; q++) {
            const double2 v = a.psi[b | soff[kk + 4 * q]];
            xr[q] = v.x;
            xi[q] = v.y;
        }
        const uint64_t b0 = __shfl_sync(0xffffffffu, b, (2 * kk) * 4);        // the lane's two output
        const uint64_t b1 = __shfl_sync(0xffffffffu, b, (2 * kk + 1) * 4);    // groups (D columns)
#pragma unroll
        for (int rt = 0; rt < D / 8; rt++) {       // output amplitudes 8 rt .. 8 rt + 7: re rows, im rows
            double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int r0 = 8 * rt + D * h;
#pragma unroll
                for (int ks = 0; ks < R / 4; ks++) {
                    const double av = sM[(r0 + n) * P + 4 * ks + kk];
                    const double bv = ks < D / 4 ? xr[ks] : xi[ks - D / 4];
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                 : "+d"(d[h][0]), "+d"(d[h][1])
                                 : "d"(av), "d"(bv));
                }
            }
            const uint64_t o = soff[8 * rt + n];
            a.psi[b0 | o] = make_double2(d[0][0], d[1][0]);
            a.psi[b1 | o] = make_double2(d[0][1], d[1][1]);
        }
    }
}

// Which dense / controlled ops take the DMMA kernel (measured, profiles/r02_op_microbench.jsonl): k = 5
// always (FP64-bound: 0.43 -> 0.55 of the HBM peak); k = 3, 4 when a target sits in the low 5 bits (the
// thread-per-group kernel then reads 2^k x 16 B per thread at a warp stride: k = 4 low 0.52 -> 0.86).
// HHLSV_JIT=dmma=0 disables it (A/B experiments).
static bool dmma_pick(const DenseArgs &a) {
    if (!jit_config().dmma || a.k < 3) return false;
    if (a.k == 5) return true;
    int lo = 64, hi = 0;
    for (int i = 0; i < a.k; i++) {
        lo = a.tpos[i] < lo ? a.tpos[i] : lo;
        hi = a.tpos[i] > hi ? a.tpos[i] : hi;
    }
    return a.k == 4 ? lo < 5 : hi < 5;          // k = 3: only when every target is low (split: a tie)
}

cudaError_t launch_dense(const DenseArgs &a, cudaStream_t s) {
    if (a.n_groups == 0) return cudaSuccess;
    if (a.k >= 3 && a.n_groups % 8 == 0 && dmma_pick(a)) {
        const uint64_t nb = a.n_groups / 8;
        switch (a.k) {
            case 3: k_dense_dmma<3><<<grid_for(nb, kThreads / 32), kThreads, 0, s>>>(a, nb); break;
            case 4: k_dense_dmma<4><<<grid_for(nb, kThreads / 32), kThreads, 0, s>>>(a, nb); break;
            case 5: k_dense_dmma<5><<<grid_for(nb, kThreads / 32), kThreads, 0, s>>>(a, nb); break;
        }
        return cudaGetLastError();
    }
    switch (a.k) {
        case 1: k_dense<1, 4><<<grid_for(a.n_groups, kThreads * 4), kThreads, 0, s>>>(a); break;
        case 2: k_dense<2, 2><<<grid_for(a.n_groups, kThreads * 2), kThreads, 0, s>>>(a); break;
        case 3: k_dense<3, 1><<<grid_for(a.n_groups, kThreads), kThreads, 0, s>>>(a); break;
        case 4: k_dense<4, 1><<<grid_for(a.n_groups, kThreads), kThreads, 0, s>>>(a); break;
        case 5: k_dense<5, 1><<<grid_for(a.n_groups, kThreads), kThreads, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ========================================================= a6 diagonal ====
__global__ void __launch_bounds__(kThreads) k_diag(const DiagArgs a) {
    extern __shared__ double2 stab[];
    for (int i = threadIdx.x; i < a.table_len; i += blockDim.x) stab[i] = a.table[i];
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 2;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * 2 + threadIdx.x; i0 < a.n_amps; i0 += stride) {
        uint64_t ii[2] = {i0, i0 + blockDim.x};
        double2 v[2];
#pragma unroll
        for (int q = 0; q < 2; q++)
            if (ii[q] < a.n_amps) v[q] = a.psi[ii[q]];
#pragma unroll
        for (int q = 0; q < 2; q++) {
            if (ii[q] >= a.n_amps) continue;
            uint32_t idx = a.gidx;
            for (int j = 0; j < a.nl; j++) idx |= (uint32_t)((ii[q] >> a.pos[j]) & 1ull) << a.tbit[j];
            a.psi[ii[q]] = cmul(stab[idx], v[q]);
        }
    }
}

cudaError_t launch_diag(const DiagArgs &a, cudaStream_t s) {
    const size_t smem = sizeof(double2) * a.table_len;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_diag<<<grid_for(a.n_amps, kThreads * 2), kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

// ======================================================= a7 recip RY ====
__global__ void __launch_bounds__(kThreads) k_recip(const RecipArgs a) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t abit = 1ull << a.anc;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.n_pairs; p += stride) {
        const uint64_t i0 = insz(p, a.anc);
        const double2 x0 = a.psi[i0], x1 = a.psi[i0 | abit];
        uint64_t m = a.mglob;
        if (a.contiguous) {
            m |= ((i0 >> a.lo) & a.lmask) << a.sh;
        } else {
            for (int j = 0; j < a.nlc; j++) m |= ((i0 >> a.lpos[j]) & 1ull) << a.lbit[j];
        }
        const double sv = recip_s(m, a.n_c, a.dL, a.is_signed, a.snap);
        const double cv = sqrt(fma(-sv, sv, 1.0));
        a.psi[i0] = make_double2(cv * x0.x - sv * x1.x, cv * x0.y - sv * x1.y);
        a.psi[i0 | abit] = make_double2(sv * x0.x + cv * x1.x, sv * x0.y + cv * x1.y);
    }
}

cudaError_t launch_recip(const RecipArgs &a, cudaStream_t s) {
    k_recip<<<grid_for(a.n_pairs, kThreads), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// ===================================================== a3 product init ====
__global__ void __launch_bounds__(kThreads) k_product(const ProductArgs a) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_amps; i += stride) {
        const uint64_t gi = a.rank_base | i;
        double2 amp = make_double2(0.0, 0.0);
        if (!(gi & a.zero_mask)) {
            amp = make_double2(1.0, 0.0);
            for (int g = 0; g < a.ngroups; g++) {
                uint32_t idx = 0;
                for (int r = 0; r < a.nruns[g]; r++)
                    idx |= (uint32_t)((gi >> a.rsrc[g][r]) & ((1ull << a.rlen[g][r]) - 1ull)) << a.rdst[g][r];
                amp = g == 0 ? __ldg(&a.tab[g][idx]) : cmul(amp, __ldg(&a.tab[g][idx]));
            }
        }
        a.psi[i] = amp;
    }
}

cudaError_t launch_product(const ProductArgs &a, cudaStream_t s) {
    k_product<<<grid_for(a.n_amps, kThreads), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

__global__ void k_zero(double2 *psi, uint64_t n, int set_first) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        psi[i] = make_double2((set_first && i == 0) ? 1.0 : 0.0, 0.0);
}

cudaError_t launch_zero_init(double2 *psi, uint64_t n, int set_first, cudaStream_t s) {
    k_zero<<<grid_for(n, kThreads), kThreads, 0, s>>>(psi, n, set_first);
    return cudaGetLastError();
}

// ======================================================= f1 tile pass ====
// Tile pass v3 (see kernels.cuh): persistent CTAs, cp.async double buffering of whole
// tiles (2^T x 16 B, XOR swizzled), op descriptors staged once per CTA in shared memory,
// a per-tile cooperative prologue (control checks + tile part of every index), and
// register-resident op phases: within a phase each thread holds the 16 amplitudes spanned by
// the phase's 4 register bits and applies every op of the phase without touching shared
// memory. ONE HBM read + write for the whole op list.
static_assert(sizeof(RegOp) % 16 == 0, "RegOp must be 16-byte sized");

__device__ __forceinline__ uint32_t swz(uint32_t u) {
    return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// deposit the bits of c into the set bits of M (constexpr; register-slot arithmetic)
__host__ __device__ constexpr int dep_mask(int c, int M) {
    int out = 0, bit = 0;
    for (int i = 0; i < 4; i++)
        if ((M >> i) & 1) {
            if ((c >> bit) & 1) out |= 1 << i;
            bit++;
        }
    return out;
}
__host__ __device__ constexpr int popc4(int M) { return (M & 1) + ((M >> 1) & 1) + ((M >> 2) & 1) + ((M >> 3) & 1); }

// Dense / controlled op whose targets are the register bits of mask M (matrix bit order =
// ascending register bits, re-ordered on the host). rcm/rcv: register-bit controls (HasC).
// Real matrices (H, V, V^T, RY — flagged by the host) use half the FP64 work.
template <int M, bool HasC, bool Real>
__device__ __forceinline__ void reg_dense(double2 (&v)[kRegAmps], const double2 *__restrict__ U, int rcm, int rcv) {
    constexpr int K = popc4(M);
    constexpr int D = 1 << K;
    if (K <= 1) {
        double2 u[D * D];
#pragma unroll
        for (int i = 0; i < D * D; i++) u[i] = __ldg(&U[i]);
#pragma unroll
        for (int g = 0; g < kRegAmps; g++) {
            if (g & M) continue;
            if (HasC && (g & rcm) != rcv) continue;
            double2 in[D];
#pragma unroll
            for (int c = 0; c < D; c++) in[c] = v[g | dep_mask(c, M)];
#pragma unroll
            for (int r = 0; r < D; r++) {
                double2 acc;
                if (Real) {
                    acc.x = u[r * D] .x * in[0].x;
                    acc.y = u[r * D].x * in[0].y;
#pragma unroll
                    for (int c = 1; c < D; c++) {
                        acc.x = fma(u[r * D + c].x, in[c].x, acc.x);
                        acc.y = fma(u[r * D + c].x, in[c].y, acc.y);
                    }
                } else {
                    acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < D; c++) cfma(acc, u[r * D + c], in[c]);
                }
                v[g | dep_mask(r, M)] = acc;
            }
        }
    } else {
#pragma unroll
        for (int g = 0; g < kRegAmps; g++) {
            if (g & M) continue;
            if (HasC && (g & rcm) != rcv) continue;
            double2 in[D];
#pragma unroll
            for (int c = 0; c < D; c++) in[c] = v[g | dep_mask(c, M)];
#pragma unroll
            for (int r = 0; r < D; r++) {
                double2 acc = make_double2(0.0, 0.0);
                if (Real) {
#pragma unroll
                    for (int c = 0; c < D; c++) {
                        const double w = __ldg(&U[r * D + c].x);
                        acc.x = fma(w, in[c].x, acc.x);
                        acc.y = fma(w, in[c].y, acc.y);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < D; c++) cfma(acc, __ldg(&U[r * D + c]), in[c]);
                }
                v[g | dep_mask(r, M)] = acc;
            }
        }
    }
}

template <int M>
__device__ __forceinline__ void reg_dense_dispatch(double2 (&v)[kRegAmps], const double2 *__restrict__ U, int rcm,
                                                   int rcv, bool real) {
    if (rcm) {
        if (real) reg_dense<M, true, true>(v, U, rcm, rcv);
        else reg_dense<M, true, false>(v, U, rcm, rcv);
    } else {
        if (real) reg_dense<M, false, true>(v, U, 0, 0);
        else reg_dense<M, false, false>(v, U, 0, 0);
    }
}

template <int A>   // A = register bit of the ancilla
__device__ __forceinline__ void reg_recip(double2 (&v)[kRegAmps], const RegOp &op, uint64_t mbase) {
    const int n_c = op.n_c, sg = op.is_signed;
    const double dL = op.dL, snap = op.snap;
#pragma unroll
    for (int j = 0; j < kRegAmps; j++) {
        if ((j >> A) & 1) continue;
        const uint64_t m = mbase | op.ridx[j];
        const double sv = recip_s(m, n_c, dL, sg, snap);
        const double cv = sqrt(fma(-sv, sv, 1.0));
        const double2 x0 = v[j], x1 = v[j | (1 << A)];
        v[j] = make_double2(cv * x0.x - sv * x1.x, cv * x0.y - sv * x1.y);
        v[j | (1 << A)] = make_double2(sv * x0.x + cv * x1.x, sv * x0.y + cv * x1.y);
    }
}

__device__ __forceinline__ uint64_t gather_runs(uint64_t x, int n, const uint8_t *src, const uint8_t *len,
                                                const uint8_t *dst) {
    uint64_t o = 0;
    for (int i = 0; i < n; i++) o |= ((x >> src[i]) & ((1ull << len[i]) - 1ull)) << dst[i];
    return o;
}

__global__ void __launch_bounds__(256) k_tile(const TileArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int T = a.T;
    const uint32_t NT = 1u << T;
    const int nthr = (int)blockDim.x;            // = NT / 16
    double2 *buf0 = reinterpret_cast<double2 *>(smem_raw);
    double2 *buf1 = buf0 + NT;
    RegOp *sops = reinterpret_cast<RegOp *>(buf1 + NT);
    const int nops = a.nops;
    uint64_t *tinfo = reinterpret_cast<uint64_t *>(sops + nops);     // per op: tile part (bit 63: skip)
    const int SA = (T + 1) / 2, SB = T - SA;
    uint64_t *depA = tinfo + nops;
    uint64_t *depB = depA + (1 << SA);
    {   // stage op descriptors (16-byte vectors)
        const int4 *src = reinterpret_cast<const int4 *>(a.ops);
        int4 *dst = reinterpret_cast<int4 *>(sops);
        const int nv = nops * (int)(sizeof(RegOp) / 16);
        for (int i = threadIdx.x; i < nv; i += nthr) dst[i] = src[i];
    }
    const uint32_t maskA = (1u << SA) - 1u;
    __shared__ int s_tbits[16];
    for (int i = threadIdx.x; i < 16; i += nthr) s_tbits[i] = a.tbits[i];
    __syncthreads();
    for (int u = threadIdx.x; u < (1 << SA); u += nthr) {
        uint64_t d = 0;
        for (int i = 0; i < SA; i++)
            if ((u >> i) & 1) d |= 1ull << s_tbits[i];
        depA[u] = d;
    }
    for (int u = threadIdx.x; u < (1 << SB); u += nthr) {
        uint64_t d = 0;
        for (int i = 0; i < SB; i++)
            if ((u >> i) & 1) d |= 1ull << s_tbits[SA + i];
        depB[u] = d;
    }

    auto tile_base = [&](uint64_t tile) {
        uint64_t b = tile;
        for (int i = 0; i < T; i++) b = insz(b, s_tbits[i]);
        return b;
    };
    auto prefetch = [&](uint64_t tile, double2 *dst) {
        const uint64_t base = tile_base(tile);
        for (uint32_t u = threadIdx.x; u < NT; u += nthr)
            cp_async16(&dst[swz(u)], &a.psi[base | depA[u & maskA] | depB[u >> SA]]);
    };
    __syncthreads();

    uint64_t tile = blockIdx.x;
    if (tile < a.n_tiles) prefetch(tile, buf0);
    cp_async_commit();
    for (int it = 0; tile < a.n_tiles; tile += gridDim.x, it++) {
        double2 *cur = (it & 1) ? buf1 : buf0;
        double2 *nxt = (it & 1) ? buf0 : buf1;
        const uint64_t next = tile + gridDim.x;
        if (next < a.n_tiles) prefetch(next, nxt);
        cp_async_commit();
        const uint64_t base = tile_base(tile);
        const uint64_t gbase = a.rank_base | base;
        // tile prologue: control check and tile part of the index of every op
        for (int i = threadIdx.x; i < nops; i += nthr) {
            const RegOp &op = sops[i];
            uint64_t t = gather_runs(gbase, op.ngr, op.g_src, op.g_len, op.g_dst);
            if ((gbase & op.gcm) != op.gcv) t |= 1ull << 63;
            tinfo[i] = t;
        }
        cp_async_wait<1>();
        __syncthreads();
        for (int p = 0; p < a.nphase; p++) {
            const RegPhase &ph = a.phases[p];
            uint32_t tb = 0;                          // tile-local index bits of this thread
            for (int i = 0; i < T - kRegBits; i++) tb |= (uint32_t)((threadIdx.x >> i) & 1) << ph.tpos[i];
            uint32_t rd[kRegAmps];
#pragma unroll
            for (int j = 0; j < kRegAmps; j++) {
                uint32_t d = 0;
#pragma unroll
                for (int i = 0; i < kRegBits; i++)
                    if ((j >> i) & 1) d |= 1u << ph.R[i];
                rd[j] = d;
            }
            double2 v[kRegAmps];
#pragma unroll
            for (int j = 0; j < kRegAmps; j++) v[j] = cur[swz(tb | rd[j])];
            for (int oi = ph.op0; oi < ph.op1; oi++) {
                const uint64_t ti = tinfo[oi];
                if (ti >> 63) continue;                                    // CTA-uniform skip
                const RegOp &op = sops[oi];
                if (op.kind == 0) {
                    if ((tb & op.tcm) != op.tcv) continue;                // thread controls
                    const double2 *U = a.blob + op.data_off;
                    const int rcm = op.rcm, rcv = op.rcv;
                    const bool real = op.is_signed != 0;      // dense ops reuse is_signed as the real flag
                    switch (op.mask) {
#define DCASE(M) case M: reg_dense_dispatch<M>(v, U, rcm, rcv, real); break;
                        DCASE(1) DCASE(2) DCASE(3) DCASE(4) DCASE(5) DCASE(6) DCASE(7) DCASE(8)
                        DCASE(9) DCASE(10) DCASE(11) DCASE(12) DCASE(13) DCASE(14) DCASE(15)
#undef DCASE
                        default: break;
                    }
                } else {
                    const uint64_t b = ti | gather_runs(tb, op.ntr, op.t_src, op.t_len, op.t_dst);
                    if (op.kind == 1) {
                        const double2 *tab = a.blob + op.data_off;
                        double2 ph_[kRegAmps];
#pragma unroll
                        for (int j = 0; j < kRegAmps; j++) ph_[j] = __ldg(&tab[(uint32_t)b | op.ridx[j]]);
#pragma unroll
                        for (int j = 0; j < kRegAmps; j++) v[j] = cmul(ph_[j], v[j]);
                    } else {
                        switch (op.mask) {
                            case 1: reg_recip<0>(v, op, b); break;
                            case 2: reg_recip<1>(v, op, b); break;
                            case 4: reg_recip<2>(v, op, b); break;
                            case 8: reg_recip<3>(v, op, b); break;
                            default: break;
                        }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < kRegAmps; j++) cur[swz(tb | rd[j])] = v[j];
            __syncthreads();
        }
        // write back (coalesced: consecutive threads -> consecutive low bits)
#pragma unroll 4
        for (uint32_t u = threadIdx.x; u < NT; u += nthr) a.psi[base | depA[u & maskA] | depB[u >> SA]] = cur[swz(u)];
        __syncthreads();
    }
    cp_async_wait<0>();
}

size_t tile_smem_bytes(int T, int nops) {
    const int SA = (T + 1) / 2, SB = T - SA;
    return 2 * sizeof(double2) * ((size_t)1 << T) + (sizeof(RegOp) + 8) * (size_t)nops +
           sizeof(uint64_t) * (((size_t)1 << SA) + ((size_t)1 << SB));
}

cudaError_t launch_tile(const TileArgs &a, cudaStream_t s) {
    const size_t smem = tile_smem_bytes(a.T, a.nops);
    const int threads = 1 << (a.T - kRegBits);
    cudaError_t e = cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)kSMs * per_sm;
    if (grid > a.n_tiles) grid = a.n_tiles;
    k_tile<<<(unsigned)grid, threads, smem, s>>>(a);
    return cudaGetLastError();
}

// ======================================================= a8 reductions ====
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block reduction of one value per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double ws[32];
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) ws[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < (int)(blockDim.x >> 5)) ? ws[l] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kThreads) k_norm2_partial(const double2 *psi, uint64_t n, uint64_t chunk,
                                                            double *partial) {
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    uint64_t hi = lo + chunk;
    if (hi > n) hi = n;
    double acc = 0.0;
    uint64_t i = lo + threadIdx.x;
    // 8 independent loads in flight per thread (the element order of the sum is unchanged)
    for (; i + 7ull * blockDim.x < hi; i += 8ull * blockDim.x) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = __ldcs(psi + i + (uint64_t)u * blockDim.x);
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc = fma(v[u].x, v[u].x, acc);
            acc = fma(v[u].y, v[u].y, acc);
        }
    }
    for (; i < hi; i += blockDim.x) {
        const double2 v = psi[i];
        acc = fma(v.x, v.x, acc);
        acc = fma(v.y, v.y, acc);
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(1024) k_sum_final(const double *partial, int np, double *out) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[i];
    acc = block_sum(acc);
    if (threadIdx.x == 0) out[0] = acc;
}

cudaError_t launch_norm2(const double2 *psi, uint64_t n, double *partial, double *out, cudaStream_t s) {
    const uint64_t chunk = (n + kRedBlocks - 1) / kRedBlocks;
    k_norm2_partial<<<kRedBlocks, kThreads, 0, s>>>(psi, n, chunk, partial);
    k_sum_final<<<1, 1024, 0, s>>>(partial, kRedBlocks, out);
    return cudaGetLastError();
}

int marginal_chunks(int nloc, int q) {
    // enough warps for the whole GPU, segments of >= 256 elements
    const int R = nloc - q;            // log2 elements per bin
    int c = 0;
    while ((q + c) < 12 + 5 && (R - c) > 8) c++;   // 2^(q+c) >= ~4k warps
    return 1 << c;
}

struct MargArgs {
    const double2 *psi;
    int nloc, q, logC;
    uint64_t Smask, Omask;
    int S[32];
    uint64_t step_dep;                 // deposit of 32 into O bits
    int O[64];
    int nO;
};

__device__ __forceinline__ uint64_t deposit_list(uint64_t x, const int *bits, int nb) {
    uint64_t d = 0;
    for (int i = 0; i < nb && x; i++, x >>= 1)
        if (x & 1ull) d |= 1ull << bits[i];
    return d;
}

__global__ void __launch_bounds__(kThreads) k_marginal(const MargArgs a, double *ws) {
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = 1ull << (a.q + a.logC);
    if (warp >= nwarps) return;
    const uint64_t v = warp >> a.logC, c = warp & ((1ull << a.logC) - 1ull);
    const int lr = a.nloc - a.q;                      // log2 elements per bin
    const uint64_t seg = 1ull << (lr - a.logC);
    const uint64_t r0 = c * seg + lane;
    double acc = 0.0;
    if (r0 < (c + 1) * seg) {
        const uint64_t sdep = deposit_list(v, a.S, a.q);
        uint64_t cur = deposit_list(r0, a.O, a.nO);
        const uint64_t cnt = seg >= 32 ? seg / 32 : 1;
        uint64_t j = 0;
        // 8 independent loads in flight per lane (the element order of the sum is unchanged)
        for (; j + 8 <= cnt; j += 8) {
            uint64_t ad[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                ad[u] = sdep | cur;
                cur = ((cur | ~a.Omask) + a.step_dep) & a.Omask;
            }
            double2 x[8];
#pragma unroll
            for (int u = 0; u < 8; u++) x[u] = __ldcs(a.psi + ad[u]);
#pragma unroll
            for (int u = 0; u < 8; u++) {
                acc = fma(x[u].x, x[u].x, acc);
                acc = fma(x[u].y, x[u].y, acc);
            }
        }
        for (; j < cnt; j++) {
            const double2 x = a.psi[sdep | cur];
            acc = fma(x.x, x.x, acc);
            acc = fma(x.y, x.y, acc);
            cur = ((cur | ~a.Omask) + a.step_dep) & a.Omask;
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) ws[warp] = acc;
}

__global__ void k_marginal_final(const double *ws, int logC, uint64_t nbins, double *out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nbins; v += stride) {
        double acc = 0.0;
        for (uint64_t c = 0; c < (1ull << logC); c++) acc += ws[(v << logC) + c];
        out[v] = acc;
    }
}

__device__ __forceinline__ double pattern_value(uint64_t seed, uint64_t i) {
    uint64_t z = (seed + 1) * 0x9E3779B97F4A7C15ull + i * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 29;
    return (double)(z >> 11);           // 53-bit integer: exact in a double
}

__global__ void k_fill_pattern(double *buf, uint64_t n, uint64_t seed, uint64_t offset) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        buf[i] = pattern_value(seed, offset + i);
}

__global__ void k_check_pattern(const double *buf, uint64_t n, uint64_t seed, uint64_t offset,
                                unsigned long long *mismatches) {
    unsigned long long bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        bad += buf[i] != pattern_value(seed, offset + i);
    if (bad) atomicAdd(mismatches, bad);
}

cudaError_t launch_fill_pattern(double *buf, uint64_t n, uint64_t seed, uint64_t offset, cudaStream_t s) {
    k_fill_pattern<<<148 * 8, 256, 0, s>>>(buf, n, seed, offset);
    return cudaGetLastError();
}

cudaError_t launch_check_pattern(const double *buf, uint64_t n, uint64_t seed, uint64_t offset,
                                 unsigned long long *mismatches, cudaStream_t s) {
    k_check_pattern<<<148 * 8, 256, 0, s>>>(buf, n, seed, offset, mismatches);
    return cudaGetLastError();
}

__global__ void k_pair_sum(const double *part, int nblocks, double *out) {
    double s0 = 0.0, s1 = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += 32) {
        s0 += part[2 * i];
        s1 += part[2 * i + 1];
    }
    for (int o = 16; o; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (threadIdx.x == 0) {
        out[0] = s0;
        out[1] = s1;
    }
}

cudaError_t launch_pair_sum(const double *part, int nblocks, double *out, cudaStream_t s) {
    k_pair_sum<<<1, 32, 0, s>>>(part, nblocks, out);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(1024) k_marginal_final_blocks(const double *ws, int logC, double *out) {
    const uint64_t v = blockIdx.x;
    const uint64_t C = 1ull << logC;
    double acc = 0.0;
    for (uint64_t c = threadIdx.x; c < C; c += blockDim.x) acc += ws[(v << logC) + c];
    acc = block_sum(acc);
    if (threadIdx.x == 0) out[v] = acc;
}

cudaError_t launch_marginal(const double2 *psi, int nloc, const int *S, int q, double *ws, double *out,
                            cudaStream_t s) {
    MargArgs a{};
    a.psi = psi;
    a.nloc = nloc;
    a.q = q;
    const int C = marginal_chunks(nloc, q);
    int logC = 0;
    while ((1 << logC) < C) logC++;
    a.logC = logC;
    for (int i = 0; i < q; i++) {
        a.S[i] = S[i];
        a.Smask |= 1ull << S[i];
    }
    a.nO = 0;
    for (int b = 0; b < nloc; b++)
        if (!((a.Smask >> b) & 1ull)) {
            a.O[a.nO++] = b;
            a.Omask |= 1ull << b;
        }
    // deposit of 32 into the O bits (used as the per-iteration stride of a lane)
    uint64_t d = 0;
    {
        uint64_t x = 32;
        for (int i = 0; i < a.nO && x; i++, x >>= 1)
            if (x & 1ull) d |= 1ull << a.O[i];
    }
    a.step_dep = d;
    const uint64_t nwarps = 1ull << (q + logC);
    const uint64_t blocks = (nwarps * 32 + kThreads - 1) / kThreads;
    k_marginal<<<(unsigned)blocks, kThreads, 0, s>>>(a, ws);
    const uint64_t nbins = 1ull << q;
    if (logC >= 8)      // many partials per bin: one block per bin (fixed-order strided sums + block tree)
        k_marginal_final_blocks<<<(unsigned)nbins, 1024, 0, s>>>(ws, logC, out);
    else
        k_marginal_final<<<grid_for(nbins, kThreads), kThreads, 0, s>>>(ws, logC, nbins, out);
    return cudaGetLastError();
}

// ============================================================ shot sampling ====
__device__ __forceinline__ uint64_t sample_phys(const SampleArgs &a, uint64_t L) {
    uint64_t P = a.lo[L & ((1ull << a.lb1) - 1ull)];
    const uint64_t hi = L >> a.lb1;
    for (int q = a.lb1; q < a.n; q++)
        if ((hi >> (q - a.lb1)) & 1ull) P |= 1ull << a.phys[q];
    return P;
}
__device__ __forceinline__ double sample_p(const SampleArgs &a, uint64_t P) {
    const double2 v = a.psi[P];
    return __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
}

// one warp per block: lanes sum strided elements sequentially, then the halving tree
__global__ void k_sample_blocks(const SampleArgs a) {
    // the low-bit offset table in shared memory: lanes index it at 32 different entries per load
    // (a by-value parameter indexed per lane would serialise in the constant cache)
    __shared__ uint64_t lo_s[1 << kSampleLB1];
    for (uint64_t i = threadIdx.x; i < (1ull << a.lb1); i += blockDim.x) lo_s[i] = a.lo[i];
    __syncthreads();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= a.nblk) return;
    const uint64_t per = 1ull << a.lb1;
    uint64_t hiP = 0;                               // physical bits of the block's high logical bits
    for (int q = a.lb1; q < a.n; q++)
        if ((warp >> (q - a.lb1)) & 1ull) hiP |= 1ull << a.phys[q];
    double r = 0.0;
    if (per >= 32) {
        for (uint64_t k = 0; k < per / 32; k++) {
            const double pv = sample_p(a, hiP | lo_s[k * 32 + lane]);
            r = k == 0 ? pv : __dadd_rn(r, pv);
        }
    } else if ((uint64_t)lane < per) {
        r = sample_p(a, hiP | lo_s[lane]);
    }
    for (int h = 16; h >= 1; h >>= 1) {
        const double o = __shfl_down_sync(0xffffffffu, r, h);
        if (lane < h) r = __dadd_rn(r, o);
    }
    if (lane == 0) a.S[warp] = r;
}

__global__ void k_sample_sup(const SampleArgs a) {
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.nsup) return;
    const uint64_t nb = 1ull << a.lb2;
    double r = a.S[c * nb];
    for (uint64_t b = 1; b < nb; b++) r = __dadd_rn(r, a.S[c * nb + b]);
    a.cum[c] = r;
}

__global__ void k_sample_prefix(const SampleArgs a) {
    double r = a.cum[0];
    for (uint64_t c = 1; c < a.nsup; c++) {
        r = __dadd_rn(r, a.cum[c]);
        a.cum[c] = r;
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_sample_draw(const SampleArgs a) {
    const uint64_t sidx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sidx >= a.shots) return;
    const double u = (double)(splitmix64(a.seed + (sidx + 1) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
    const double total = a.cum[a.nsup - 1];
    const double t = __dmul_rn(u, total);
    // superblock: first c with cum_c > t (binary search on the non-decreasing prefix)
    uint64_t lo = 0, hi = a.nsup;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a.cum[mid] > t) hi = mid;
        else lo = mid + 1;
    }
    uint64_t c = lo;
    if (c >= a.nsup) {                              // rounding: last superblock with a nonzero sum
        c = a.nsup - 1;
        while (c > 0 && a.cum[c] == a.cum[c - 1]) c--;
    }
    // block inside the superblock
    const uint64_t nb = 1ull << a.lb2;
    double r = c ? a.cum[c - 1] : 0.0;
    uint64_t blk = UINT64_MAX, lastnz = c * nb;
    double before = r, before_lastnz = r;
    for (uint64_t b = c * nb; b < (c + 1) * nb; b++) {
        const double nr = __dadd_rn(r, a.S[b]);
        if (a.S[b] > 0.0) { lastnz = b; before_lastnz = r; }
        if (nr > t) { blk = b; before = r; break; }
        r = nr;
    }
    if (blk == UINT64_MAX) { blk = lastnz; before = before_lastnz; }
    // element inside the block (logical order)
    const uint64_t per = 1ull << a.lb1;
    uint64_t hiP = 0;
    for (int q = a.lb1; q < a.n; q++)
        if ((blk >> (q - a.lb1)) & 1ull) hiP |= 1ull << a.phys[q];
    r = before;
    uint64_t el = UINT64_MAX, lastel = 0;
    for (uint64_t i = 0; i < per; i++) {
        const double pv = sample_p(a, hiP | a.lo[i]);
        const double nr = __dadd_rn(r, pv);
        if (pv > 0.0) lastel = i;
        if (nr > t) { el = i; break; }
        r = nr;
    }
    if (el == UINT64_MAX) el = lastel;
    a.out[sidx] = (blk << a.lb1) | el;
}

cudaError_t launch_sample_sums(const SampleArgs &a, cudaStream_t s) {
    const uint64_t threads = a.nblk * 32;
    k_sample_blocks<<<(unsigned)((threads + kThreads - 1) / kThreads), kThreads, 0, s>>>(a);
    k_sample_sup<<<(unsigned)((a.nsup + kThreads - 1) / kThreads), kThreads, 0, s>>>(a);
    k_sample_prefix<<<1, 1, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sample_draw(const SampleArgs &a, cudaStream_t s) {
    if (a.shots == 0) return cudaSuccess;
    k_sample_draw<<<(unsigned)((a.shots + kThreads - 1) / kThreads), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// ======================================================= gather / scatter ====
__global__ void k_gather(const GatherArgs a) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.count; e += stride) {
        uint64_t L;
        if (a.nfree == 0) {
            L = a.first + e;
        } else {
            L = a.fixed;
            uint64_t x = a.first + e;
            for (int i = 0; i < a.nfree; i++)
                if ((x >> i) & 1ull) L |= 1ull << a.free_q[i];
        }
        uint64_t P = 0;
        for (int q = 0; q < a.n; q++)
            if ((L >> q) & 1ull) P |= 1ull << a.phys[q];
        double2 v = make_double2(0.0, 0.0);
        if ((P >> a.nloc) == a.rank) v = a.psi[P & ((1ull << a.nloc) - 1ull)];
        a.out[e] = v;
    }
}

cudaError_t launch_gather(const GatherArgs &a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    k_gather<<<grid_for(a.count, kThreads), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

__global__ void k_scatter(const ScatterArgs a) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.count; e += stride) {
        const uint64_t L = a.first + e;
        uint64_t P = 0;
        for (int q = 0; q < a.n; q++)
            if ((L >> q) & 1ull) P |= 1ull << a.phys[q];
        if ((P >> a.nloc) == a.rank) a.psi[P & ((1ull << a.nloc) - 1ull)] = a.in[e];
    }
}

cudaError_t launch_scatter(const ScatterArgs &a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    k_scatter<<<grid_for(a.count, kThreads), kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// ====================================================== K7 pack / unpack ====
__global__ void k_pack(const double2 *psi, double2 *buf, int lbit, int val, uint64_t off, uint64_t cnt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride)
        buf[j] = psi[insz(off + j, lbit) | ((uint64_t)val << lbit)];
}
__global__ void k_unpack(double2 *psi, const double2 *buf, int lbit, int val, uint64_t off, uint64_t cnt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride)
        psi[insz(off + j, lbit) | ((uint64_t)val << lbit)] = buf[j];
}

// Multi-bit form (multi-qubit exchanges): element j of the slot whose bits L (ascending, nl <= 8)
// equal `pat` (bit i of pat <- L[i]) is psi[deposit(off + j) | pat bits], deposit = zeros inserted at L.
struct PatBits {
    int nl;
    int L[8];
    uint64_t patmask;
};
__device__ __forceinline__ uint64_t pat_index(const PatBits &b, uint64_t x) {
    for (int i = 0; i < b.nl; i++) x = insz(x, b.L[i]);
    return x | b.patmask;
}
__global__ void k_packm(const double2 *psi, double2 *buf, PatBits b, uint64_t off, uint64_t cnt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride)
        buf[j] = psi[pat_index(b, off + j)];
}
__global__ void k_unpackm(double2 *psi, const double2 *buf, PatBits b, uint64_t off, uint64_t cnt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride)
        psi[pat_index(b, off + j)] = buf[j];
}
static PatBits pat_bits(const int *L, int nl, uint32_t pat) {
    PatBits b{};
    b.nl = nl;
    for (int i = 0; i < nl; i++) b.L[i] = L[i];
    for (int i = 0; i < nl; i++)
        if ((pat >> i) & 1) b.patmask |= 1ull << L[i];
    return b;
}
cudaError_t launch_pack_multi(const double2 *psi, double2 *buf, const int *L, int nl, uint32_t pat, uint64_t off,
                              uint64_t cnt, cudaStream_t s) {
    if (nl < 1 || nl > 8) return cudaErrorInvalidValue;
    k_packm<<<grid_for(cnt, kThreads), kThreads, 0, s>>>(psi, buf, pat_bits(L, nl, pat), off, cnt);
    return cudaGetLastError();
}
cudaError_t launch_unpack_multi(double2 *psi, const double2 *buf, const int *L, int nl, uint32_t pat, uint64_t off,
                                uint64_t cnt, cudaStream_t s) {
    if (nl < 1 || nl > 8) return cudaErrorInvalidValue;
    k_unpackm<<<grid_for(cnt, kThreads), kThreads, 0, s>>>(psi, buf, pat_bits(L, nl, pat), off, cnt);
    return cudaGetLastError();
}

cudaError_t launch_pack(const double2 *psi, double2 *buf, int lbit, int val, uint64_t off, uint64_t cnt,
                        cudaStream_t s) {
    k_pack<<<grid_for(cnt, kThreads), kThreads, 0, s>>>(psi, buf, lbit, val, off, cnt);
    return cudaGetLastError();
}
cudaError_t launch_unpack(double2 *psi, const double2 *buf, int lbit, int val, uint64_t off, uint64_t cnt,
                          cudaStream_t s) {
    k_unpack<<<grid_for(cnt, kThreads), kThreads, 0, s>>>(psi, buf, lbit, val, off, cnt);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace hhlsv
