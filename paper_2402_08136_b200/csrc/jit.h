// NVRTC specialisation of tile passes (see jit.cpp).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kernels.cuh"

namespace hhlsv {

struct JitPass {
    std::string name;
    std::string src;
    cudaKernel_t kern = nullptr;
    size_t smem_extra = 0;     // total dynamic shared memory of the generated kernel (bytes)
    int nthr = 256;            // threads per CTA = 2^(T - register bits)
    // wide (>= 3-target) dense matrices read as constant-bank operands: (blob offset, entries) in
    // the order of the kernel's by-value parameter cwa (<= 32 KB of kernel parameters: per-launch,
    // hence coherent even when passes with identical structure share one cached module), and the
    // host copy of those values passed at every launch
    std::vector<std::pair<uint64_t, uint64_t>> cwide;
    std::vector<double2> cwvals;
    // launch configuration, resolved on the first launch (attribute + occupancy queries are host
    // work a launch-bound small program should not repeat)
    mutable int per_sm = 0, sms = 0;
    // fused marginal (TileArgs::red >= 0): device buffer of 2 doubles per CTA of the launch grid
    double *red = nullptr;
};

// Product-state init fused into the first tile pass: the pass computes its tile's amplitudes
// (prod_g table_g[gather_g(global index)], 0 where a zero_mask bit is set) instead of reading them.
struct InitSpec {
    uint64_t zero_mask = 0;
    std::vector<size_t> off;                 // per group: blob offset of its table
    std::vector<std::vector<int>> bits;      // per group: physical bits, table bit j <- bits[j]
};

// Code-generation switches of the tile JIT (all default on / measured best). Developer A/B
// experiments only: parsed ONCE from HHLSV_JIT="key=value,..." (e.g. HHLSV_JIT=pf=0,group=0).
struct JitConfig {
    bool direct = true;       // direct: HBM <-> register first/last phases when the thread bits are coalesced
    bool prefetch = true;     // pf: L2 prefetch of the CTA's next tile at the top of each tile
    int pf_dist = 1;          // pfdist: prefetch distance in tiles
    bool group = true;        // group: consecutive diagonal ops of a phase share per-slot factor products
    bool rtab = true;         // rtab: per-tile (s_m, c_m) tables of the reciprocal rotation
    bool hoist = true;        // hoist: phase p+1's sub-tables are built at the end of phase p
    bool sparse = true;       // sparse: exact structural zeros of wide matrices skipped at codegen
    bool tail = true;         // tail: a trailing wide dense op writes straight into the store buffer
    bool cw = true;           // cw: >= 3-target matrices as by-value kernel parameters (constant bank)
    bool ctab = true;         // ctab: small diagonal tables (no out-of-tile index bits, <= 2 thread bits) too
    int ctab_bits = 2;        // ctabbits: max thread bits of a constant-bank table index (selected per thread)
    int nbuf = 1;             // nbuf: 1 single tile buffer (occupancy), 2 cp.async double buffering
    int min_blocks = 0;       // minb: __launch_bounds__ min blocks per SM (0 = from shared memory)
    int reg_bits = 4;         // rb: register bits per phase (4: 16 amplitudes per thread, 3: 8)
    bool graphs = true;       // graphs: small single-rank programs replay a captured CUDA graph
    bool xoverlap = true;     // xoverlap: a pass followed by a top-bit exchange is split by slot and pipelined
    bool skeleton = false;    // skeleton: TIMING EXPERIMENT (wrong results): passes move data, apply no op
    int ru = 0;               // ru: rows per block of the rolled wide-op loop (0 = 16 real / 2 complex)
    bool smem_clobber = false;  // clobber: "memory" clobber on every shared-memory asm access
    std::string ptxas_opt = "-Xptxas=-O3";   // ptxas: optimisation level passed to NVRTC's ptxas
    // scheduler / front-end switches (same variable)
    int wmin = 3;             // wmin: low physical bits every tile holds (3 = 128-byte segments)
    int diag_merge = -1;      // dmerge: in-phase diagonal merge width (-1 = CompileOptions::diag_merge)
    int eigen_chunk = 0;      // echunk: clock bits per eigen-phase table (0 = front-end default)
    bool init_fuse = true;    // initfuse: product-state init computed inside the first tile pass
    bool mred = true;         // mred: the last tile pass accumulates the HHL ancilla marginal (fused readout)
    bool spillfb = true;      // spillfb: regenerate a spilling pass with the JitVariant fallbacks
    bool twiddle = true;      // twiddle: a diagonal's x1 multiplies folded into the following butterfly
    bool dmma = true;         // dmma: streaming dense k = 5 / low-target k = 3, 4 on the FP64 tensor cores
    bool wrun = true;         // wrun: per-tile products of runs of 4-qubit ops on a phase's register bits
    bool vdmma = false;       // vdmma: a last phase holding one real 4-qubit op (V) on the FP64 tensor cores
                              //        (correct, measured slower: DESIGN §6.2)
    int dalap = 0;            // dalap: the first N tile passes defer their diagonal ops (as late as possible;
                              //        measured slower: profiles/r02_experiments.txt)
};
const JitConfig &jit_config();

// Per-pass code-generation fallbacks (program_create retries a pass whose ptxas output spills with
// these, keeping the variant that spills least): both trade a little FP64 / load work for registers.
struct JitVariant {
    bool no_ctab = false;      // diagonal tables from L1 (__ldg) instead of per-thread selects of kernel params
    bool no_group = false;     // no shared per-slot factor products across a phase's diagonal ops
};

bool jit_available(std::string *why);
std::string gen_tile_kernel(const std::string &name, const dev::TileArgs &a, const std::vector<dev::RegPhase> &ph,
                            const std::vector<dev::RegOp> &ops, size_t *smem_extra = nullptr,
                            const InitSpec *init = nullptr,
                            std::vector<std::pair<uint64_t, uint64_t>> *cwide = nullptr,
                            const std::vector<double2> *hblob = nullptr,    // host blob: structural zeros
                            const JitVariant &var = JitVariant());
// ptxas spill-store bytes of a generated pass (compiles it once; the cubin is kept for jit_build /
// jit_compile_only). -1 if the compilation fails (jit_build then reports the error).
int jit_spill_bytes(const std::string &src);
// The spill bytes of a source already probed in this process (no compilation); false if unknown.
bool jit_spill_cached(const std::string &src, int *spill);
void jit_build(std::vector<JitPass> &passes);            // compile (cached) + load; throws on failure
std::vector<char> jit_compile_only(const std::string &src, std::string &err);
// Name under which HHLSV_JIT_DUMP stores a pass's full source ("tile_<hash>"), for debug tooling.
std::string jit_source_tag(const std::string &src);
// Launch tiles [tile0, n_tiles) of a pass (tile0 = 0: the whole pass).
cudaError_t jit_launch(const JitPass &p, double2 *psi, const double2 *blob, uint64_t n_tiles, uint64_t rank_base,
                       int T, cudaStream_t s, uint64_t tile0 = 0);
// CTAs jit_launch uses for tiles [0, n_tiles) (after the pass's first launch resolved its occupancy).
uint64_t jit_grid(const JitPass &p, uint64_t n_tiles);
size_t jit_smem_bytes(int T, size_t extra);

}  // namespace hhlsv
