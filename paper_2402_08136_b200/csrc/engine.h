// Device state and resident programs (internal).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "comm.h"
#include "jit.h"
#include "kernels.cuh"
#include "sv_internal.h"

struct sv_state {
    int n = 0;              // total qubits
    int g = 0;              // global (rank) qubits = log2(world)
    int nloc = 0;           // local qubits
    int world = 1, rank = 0, device = 0;
    cudaStream_t stream = nullptr;
    double2 *psi = nullptr; // 2^nloc local amplitudes, physical order
    std::vector<int> phys;  // logical qubit -> physical bit
    // workspace
    double *d_red = nullptr;        // reduction partials
    size_t red_len = 0;
    double *d_scalar = nullptr;     // 8 doubles
    double2 *d_io = nullptr;        // staging for gathers/exchanges
    size_t io_len = 0;              // in double2
    double2 *d_xsend = nullptr, *d_xrecv = nullptr;  // exchange buffers
    size_t x_len = 0;
    cudaStream_t comm_stream = nullptr;              // pipelined exchanges (created on first use)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    hhlsv::Comm comm;
    // virtual sharding (world > 1 without an NCCL id): all shards in this process on one GPU,
    // one view per virtual rank, exchanges by device copies (tests the rank-dependent paths)
    int vworld = 1;
    std::vector<sv_state *> views;
    uint64_t local_amps() const { return 1ull << nloc; }
};

namespace hhlsv {

struct LaunchRec {
    StepKind kind;
    bool skip = false;                // controlled op whose global controls do not match this rank
    dev::DenseArgs dense{};
    dev::DiagArgs diag{};
    dev::RecipArgs recip{};
    dev::ProductArgs prod{};
    dev::TileArgs tile{};
    std::vector<int> xg, xl;          // exchange: physical global bits xg[i] <-> local bits xl[i]
    int jit = -1;                     // tile: index into sv_program::jit (specialised kernel) or -1
    double flops = 0;                 // FP64 flops the launch must execute (structure-aware count)
    double bytes = 0;
};

}  // namespace hhlsv

struct sv_program {
    sv_state *sv = nullptr;
    hhlsv::Schedule sched;
    std::vector<int> phys_in;
    bool resets = false;              // starts with an initialisation step
    double2 *d_blob = nullptr;
    hhlsv::dev::RegOp *d_ops = nullptr;
    hhlsv::dev::RegPhase *d_phases = nullptr;
    std::vector<hhlsv::LaunchRec> recs;
    uint64_t n_logical = 0;
    std::vector<double2 *> d_tabs;    // product-init tables (owned)
    double h2d_bytes = 0;             // uploaded at creation
    std::vector<hhlsv::JitPass> jit;  // specialised tile passes
    std::vector<sv_program *> subs;   // virtual sharding: one program per view
    bool timing = false;
    std::vector<cudaEvent_t> ev;      // 2 per rec when timing
    // small single-rank programs replay a CUDA graph of their launches (captured on the 2nd run)
    int runs = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaStream_t gstream = nullptr;
    cudaEvent_t gev_a = nullptr, gev_b = nullptr;
    // fused marginal of the last tile pass (CompileOptions::red_qubit): per-CTA partials, then
    // d_mred[2 * kMredCtas + {0, 1}] = P(qubit = 0 / 1) after every run; nullptr = not fused
    double *d_mred = nullptr;
    static constexpr int kMredCtas = 148 * 32;
    uint64_t launches() const;
};

namespace hhlsv {
void cuda_check(cudaError_t e, const char *what);
sv_state *state_create(int n, const sv_dist *dist, cudaStream_t stream, bool zero_init = true);
void state_destroy(sv_state *sv);
// Release device memory the library's pool caches for reuse (device < 0: every device), keeping `keep` bytes.
void pool_trim(int device, size_t keep);
void state_reset(sv_state *sv);
sv_program *program_create(sv_state *sv, const std::vector<Gate> &ops, const std::vector<ProductFactor> *init,
                           const CompileOptions &co, uint64_t n_logical);
void program_run(sv_state *sv, sv_program *p);
void program_destroy(sv_program *p);
void lower_tile_step(const Step &st, dev::TileArgs &a, std::vector<double2> &blob, std::vector<dev::RegOp> &rops,
                     std::vector<dev::RegPhase> &phases, size_t &ph0_out, size_t &opbase_out, bool butterflies,
                     double prescale);
bool is_butterfly(const Gate &g, double *a);
void program_timings(sv_program *p, float *ms, int *kind, double *bytes, double *flops, int *launches, size_t cap,
                     size_t *n_out);
void state_read(sv_state *sv, uint64_t first, uint64_t count, double *out);
void state_write(sv_state *sv, uint64_t first, uint64_t count, const double *in);
double state_norm2(sv_state *sv);
void state_probabilities(sv_state *sv, const int *qubits, int nq, double *out);
// Shot sampling: `shots` logical indices drawn from |a|^2, deterministic in seed.
void state_sample(sv_state *sv, uint64_t shots, uint64_t seed, uint64_t *out);
void state_postselect(sv_state *sv, const int *fq, const int *fv, int nfixed, double *amps, uint64_t *idx,
                      uint64_t n_out, double *prob);
}  // namespace hhlsv
