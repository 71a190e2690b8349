// Kernel parameter blocks and launchers for the sm_100a state-vector kernels.
// All amplitude arrays are interleaved complex128 (double2), PHYSICAL local order.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace hhlsv {
namespace dev {

constexpr int kMaxIns = 26;      // zero-insertion bits (targets + local controls)
constexpr int kMaxDiag = 12;
constexpr int kMaxClock = 62;
constexpr int kMaxTileOps = 4096;

struct DenseArgs {               // a4/a5: dense or controlled fused gate, one streaming pass
    double2 *psi;
    uint64_t n_groups;           // 2^(nloc - k - #local controls)
    int nins;
    int ins[kMaxIns];            // sorted bits where zeros are inserted (targets + local controls)
    uint64_t cset;               // OR-mask of local control bits required to be 1
    int k;
    int tpos[5];                 // target bits, tpos[0] = LSB of the matrix index
    const double2 *U;            // 2^k x 2^k row-major, device
};

struct DiagArgs {                // a6: diagonal fused gate (phase table over <= 12 qubits)
    double2 *psi;
    uint64_t n_amps;
    int nl;                      // local table qubits
    int pos[kMaxDiag];           // physical local bit of local table qubit j
    int tbit[kMaxDiag];          // table-index bit it feeds
    uint32_t gidx;               // table-index bits from global qubits (rank)
    const double2 *table;
    int table_len;
};

struct RecipArgs {               // a7: eigenvalue-inversion RY, multiplexed by the clock register
    double2 *psi;
    uint64_t n_pairs;            // 2^(nloc-1)
    int anc;                     // ancilla physical (local) bit
    int nlc;                     // local clock bits
    int lpos[kMaxClock];         // physical bit of local clock qubit
    int lbit[kMaxClock];         // register bit it feeds
    uint64_t mglob;              // register bits from global clock qubits
    int n_c;
    double dL;                   // delta * 2^(n_c - signed) (exact)
    double snap;
    int is_signed;
    int contiguous;              // local clock bits are physical lo..lo+nlc-1 feeding register bits sh..
    int lo, sh;
    uint64_t lmask;
};

struct ProductArgs {             // a3: product-state initialisation (+ folded leading diagonals)
    double2 *psi;
    uint64_t n_amps;
    uint64_t rank_base;          // rank << nloc (global index of local 0)
    uint64_t zero_mask;          // global-index bits that must be 0 (qubits no product factor covers)
    int ngroups;                 // amplitude = prod_g tab_g[index_g(global index)]
    int nruns[4];                // index_g = OR over runs of ((gi >> src) & (2^len - 1)) << dst
    uint8_t rsrc[4][16], rlen[4][16], rdst[4][16];
    const double2 *tab[4];       // group tables (<= 2^14 entries, L2-resident)
};

// Tile pass v2: a CTA holds 2^T amplitudes of one tile in shared memory
// (cp.async double-buffered, persistent CTAs); the pass's ops are grouped in register phases:
// in phase p every thread holds the 16 amplitudes spanned by the 4 tile positions R[p] (the
// "register bits") at its own thread-bit coordinates, and applies all the phase's ops in
// registers. Phases exchange data through shared memory.
constexpr int kRegBits = 4;
constexpr int kRegAmps = 1 << kRegBits;

struct alignas(16) RegOp {       // staged in shared memory by every CTA
    int kind;                    // 0 dense/controlled, 1 diagonal, 2 recip
    int mask;                    // dense: register-bit mask of the targets; recip: 1 << (anc register bit)
    int rcm, rcv;                // dense: register-bit controls (mask / required values)
    uint32_t tcm, tcv;           // dense: controls on thread-held tile positions (tile-local masks)
    uint64_t gcm, gcv;           // controls outside the tile (global index bits): op skipped unless match
    uint32_t ridx[kRegAmps];     // diag/recip: register-slot part of the table index / clock value
    int ntr, ngr;                // bit runs: thread part (tile-local positions), tile part (global index)
    uint8_t t_src[12], t_len[12], t_dst[12];
    uint8_t g_src[48], g_len[48], g_dst[48];
    int n_c, is_signed;
    double dL, snap;
    uint64_t data_off;           // matrix (register-bit order) / table offset in the blob (double2 units)
};

struct RegPhase {
    int R[kRegBits];             // tile positions held in registers (ascending)
    int tpos[16];                // the other T - 4 tile positions (ascending) = thread bits
    int op0, op1;                // ops [op0, op1)
};

struct TileArgs {
    double2 *psi;
    uint64_t n_tiles;            // 2^(nloc - T)
    int T;
    int nreg = 4;                // register bits per phase (JIT passes: 3 or 4; the interpreter: 4)
    int tbits[16];               // sorted physical local bits of the tile
    int nphase;
    const RegPhase *phases;      // device
    int nops;                    // ops of this step (all phases)
    const RegOp *ops;            // device, this step's ops (phase op0/op1 index into it)
    const double2 *blob;         // program data blob
    uint64_t rank_base;
    // Lazy zero qubits (JIT passes only, DESIGN.md §6 "Known-zero qubits"): physical bits whose
    // amplitudes are known to be 0 when the bit is 1 (e.g. the HHL ancilla before the reciprocal
    // rotation). Out-of-tile such bits that stay zero through the pass are skipped: tiles with the
    // bit set are neither read nor written (n_tiles excludes them). Tile positions in zload are 0
    // on input (not read); tile positions in zstore are still 0 on output (not written).
    int nskip;
    int skip[8];
    uint32_t zload, zstore;
    // Out-of-tile bits mapped to the TOP of the tile index (ascending): with the exchange that follows
    // the pass on these local bits, tiles [p 2^nlow, (p+1) 2^nlow) are exactly exchange slot p
    // (pipelined pass + exchange). nlift = 0: plain ascending mapping.
    int nlift = 0;
    int lift[8];
    // Fused readout (JIT passes only): physical bit whose marginal the pass accumulates while it stores
    // the final amplitudes (per-CTA partials Σ|a|² for bit = 0 / 1, DESIGN.md §6 "Fused marginal");
    // -1 = none.
    int red = -1;
};

// ---- launchers (stream-ordered, no sync) ----
cudaError_t launch_dense(const DenseArgs &a, cudaStream_t s);
cudaError_t launch_diag(const DiagArgs &a, cudaStream_t s);
cudaError_t launch_recip(const RecipArgs &a, cudaStream_t s);
cudaError_t launch_product(const ProductArgs &a, cudaStream_t s);
cudaError_t launch_zero_init(double2 *psi, uint64_t n, int set_first, cudaStream_t s);
cudaError_t launch_tile(const TileArgs &a, cudaStream_t s);
size_t tile_smem_bytes(int T, int nops);

// Deterministic reductions. partial has >= kRedBlocks doubles; result written to out (device).
constexpr int kRedBlocks = 1184;   // 148 SMs x 8
// Fixed-order sum of nblocks (bit 0, bit 1) partial pairs written by a tile pass with a fused marginal:
// out[0] = Σ part[2i], out[1] = Σ part[2i + 1] (one warp; lane-strided then a shuffle tree).
cudaError_t launch_pair_sum(const double *part, int nblocks, double *out, cudaStream_t s);
// Seeded test pattern for transport checks: buf[i] = f(seed, offset + i) (exactly representable);
// check counts the doubles of buf that differ from the pattern into *mismatches (atomic u64).
cudaError_t launch_fill_pattern(double *buf, uint64_t n, uint64_t seed, uint64_t offset, cudaStream_t s);
cudaError_t launch_check_pattern(const double *buf, uint64_t n, uint64_t seed, uint64_t offset,
                                 unsigned long long *mismatches, cudaStream_t s);
cudaError_t launch_norm2(const double2 *psi, uint64_t n, double *partial, double *out, cudaStream_t s);
// Marginal over physical bits S (q = |S| <= 26, bit j of v <- S[j]); others O = remaining local bits.
// Writes 2^q doubles to out (device). ws must hold 2^q * C doubles (C returned by marginal_chunks).
int marginal_chunks(int nloc, int q);
cudaError_t launch_marginal(const double2 *psi, int nloc, const int *S, int q, double *ws, double *out,
                            cudaStream_t s);
// Gather amplitudes by LOGICAL index: for e < count, logical index L = fixed | deposit(first+e into free bits)
// (free = NULL: L = first + e). Physical global index via phys[]; elements not owned by rank -> 0.
struct GatherArgs {
    const double2 *psi;
    double2 *out;
    uint64_t count;
    uint64_t first;
    int n;
    int nloc;
    uint64_t rank;
    int phys[64];
    int nfree;                   // 0 -> contiguous logical range
    int free_q[64];              // free logical qubits ascending (postselect)
    uint64_t fixed;              // logical bits of fixed qubits
};
cudaError_t launch_gather(const GatherArgs &a, cudaStream_t s);
struct ScatterArgs {             // inverse of gather (sv_write): only owned elements are written
    double2 *psi;
    const double2 *in;
    uint64_t count, first;
    int n, nloc;
    uint64_t rank;
    int phys[64];
};
cudaError_t launch_scatter(const ScatterArgs &a, cudaStream_t s);
// Shot sampling (sv_sample; SPEC `sample`, Fig. 3 "10,000 measurements"): inverse-CDF draws in
// LOGICAL index order with a fixed summation order shared with the oracle:
//  p_i = re*re + im*im (two roundings + one, no FMA);
//  block b (2^lb1 logical indices): lane l of a warp sums p_{b,32k+l} for k = 0.. sequentially, then the
//    32 lane sums are combined by halving (a[j] += a[j+h], h = 16, 8, .., 1) -> S_b;
//  superblock c (2^lb2 blocks): T_c = sequential sum of its S_b; cum_c = sequential inclusive prefix;
//  shot s: u = (splitmix64(seed + (s+1)*golden) >> 11) * 2^-53, t = u * cum_last; c = first with cum_c > t;
//    running r from cum_{c-1} over the superblock's S_b -> first block with r > t; running r from the value
//    before that block over its p_i (logical order) -> first i with r > t; when rounding leaves no such
//    block / element, the last one with a nonzero sum is taken.
constexpr int kSampleLB1 = 10, kSampleLB2 = 10;
struct SampleArgs {
    const double2 *psi;
    int n, lb1, lb2;
    uint64_t nblk, nsup;
    uint64_t lo[1 << kSampleLB1];    // physical offset of the low lb1 logical bits (identity-free map)
    int phys[64];
    double *S, *cum;                 // nblk block sums, nsup superblock prefix sums (device)
    uint64_t shots, seed;
    uint64_t *out;                   // shots logical indices (device)
};
cudaError_t launch_sample_sums(const SampleArgs &a, cudaStream_t s);   // S, then cum
cudaError_t launch_sample_draw(const SampleArgs &a, cudaStream_t s);
// Exchange helpers: pack/unpack the half of the local state whose bit lbit == val, elements [off, off+cnt).
cudaError_t launch_pack(const double2 *psi, double2 *buf, int lbit, int val, uint64_t off, uint64_t cnt,
                        cudaStream_t s);
cudaError_t launch_unpack(double2 *psi, const double2 *buf, int lbit, int val, uint64_t off, uint64_t cnt,
                          cudaStream_t s);
// Multi-qubit exchanges: pack/unpack elements [off, off+cnt) of the slot whose local bits L
// (ASCENDING, nl <= 8) equal pattern pat (bit i of pat <- L[i]), in increasing order of the other bits.
cudaError_t launch_pack_multi(const double2 *psi, double2 *buf, const int *L, int nl, uint32_t pat, uint64_t off,
                              uint64_t cnt, cudaStream_t s);
cudaError_t launch_unpack_multi(double2 *psi, const double2 *buf, const int *L, int nl, uint32_t pat, uint64_t off,
                                uint64_t cnt, cudaStream_t s);

}  // namespace dev
}  // namespace hhlsv
