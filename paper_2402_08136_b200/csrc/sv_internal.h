// Internal types of the B200 HHL state-vector engine (not part of the C ABI).
//
// Layers:
//   frontend.cpp  HHL builder (Fig. 5) + fusion pass (Fig. 4)
//   compile.cpp   scheduler: logical fused ops -> physical steps (relabel SWAPs, shard
//                 exchanges, shared-memory tile passes)
//   kernels.cu    sm_100a kernels: init, dense/controlled, diagonal, reciprocal RY,
//                 tile pass, reductions, pack/unpack
//   engine.cu     device state, program execution, readout
//   comm.cpp      NCCL (dlopen'ed) pairwise exchange for global-qubit swaps
//   api.cpp       the extern "C" boundary of include/sv.h
#pragma once

#include <cstdint>
#include <complex>
#include <string>
#include <vector>

#include "sv.h"

namespace hhlsv {

using cplx = std::complex<double>;

// ------------------------------------------------------------------ gate IR ----
enum class Kind : int { Dense = SV_DENSE, Controlled = SV_CONTROLLED, Diagonal = SV_DIAGONAL,
                        RecipRY = SV_RECIP_RY, Swap = SV_SWAP };

struct Gate {
    Kind kind = Kind::Dense;
    std::vector<int> targets;      // targets[0] = LSB of the matrix index
    std::vector<int> controls;     // Controlled: controls; RecipRY: clock register LSB first
    uint64_t cvals = 0;            // bit i = required value of controls[i]
    std::vector<cplx> data;        // Dense/Controlled: 2^k x 2^k row-major; Diagonal: 2^k
    double delta = 0.0;            // RecipRY
    int is_signed = 1;
    double snap = 0.0;
};

// Algorithmic bytes of one fused op on an n-qubit state.
double alg_bytes(const Gate &g, int n);

// ------------------------------------------------------------- error status ----
struct Error {
    sv_status code;
    std::string msg;
};
[[noreturn]] void fail(sv_status code, const std::string &msg);
// Developer stage timer: with HHLSV_PROFILE=1 in the environment prints "<stage> <ms>" to stderr.
void prof_mark(const char *stage);
bool prof_on();

// Validation of one ABI gate -> internal Gate (copies the data).
Gate gate_from_abi(const sv_gate &g, int n_qubits);

// --------------------------------------------------------------- front end ----
struct HHLPlanHost {
    int n_orig = 0, N = 0, n_b = 0, n_c = 0, n = 0;
    std::vector<double> A;           // padded N x N
    std::vector<double> b_hat;       // padded, normalised
    double b_norm = 0.0;
    std::vector<double> lam;         // eigenvalues (ascending)
    std::vector<double> V;           // eigenvectors, column-major V[i + N*s]
    double lam_min = 0, lam_max = 0, kappa = 0, delta = 0, t = 0;
    std::vector<double> phi;         // phi_s = (lam_s/lam_min)(delta/2)
    double snap = 1e-5;
    int x_offset = 0;                // Hermitian embedding: x is the lower half
};

// eig_lam / eig_V (optional, both or neither): caller-supplied eigendecomposition of the padded
// matrix (hhl_options.eig_*; V row-major, column s <-> eig_lam[s]) instead of jacobi_eigh.
HHLPlanHost hhl_plan(const double *A, const double *b, int N, int clock_qubits, double snap,
                     const double *eig_lam = nullptr, const double *eig_V = nullptr);
std::vector<Gate> hhl_build(const HHLPlanHost &p, int qpe_mode = 0);
void jacobi_eigh(int N, std::vector<double> A, std::vector<double> &lam, std::vector<double> &V);

struct FuseOptions {
    int kmax = 4;          // dense/controlled target cap after fusion (0 = none)
    int diag_kmax = 10;    // diagonal width cap
    int mode = 0;          // 0: greedy structure-preserving window (B200 mode); 1: the paper's Fig. 4 fusion
};
std::vector<Gate> fuse(const std::vector<Gate> &in, const FuseOptions &o);
// cur <- nx * cur for two diagonal ops when their union has <= diag_kmax qubits (else false).
bool merge_diagonal(Gate &cur, const Gate &nx, int diag_kmax);

// Product-state prefix: if the circuit starts (from |0...0>) with gates on disjoint
// qubit sets, each a Dense gate acting on qubits untouched before, the state after
// that prefix is  (x)_f U_f|0>. Returns the number of gates folded.
struct ProductFactor {
    std::vector<int> qubits;      // logical qubits, qubits[0] = LSB of the factor index
    std::vector<cplx> vec;        // 2^|qubits| amplitudes (= column 0 of the factor's matrix)
    bool diag = false;            // a diagonal gate applied after the product state (vec = its table)
};
size_t fold_product_prefix(const std::vector<Gate> &gates, int n, std::vector<ProductFactor> &factors,
                           bool fold_diagonals = true);

// ---------------------------------------------------------------- program ----
enum class StepKind : int { InitZero, InitProduct, Dense, Diagonal, RecipRY, Tile, Exchange };

// One tile-local op inside a Tile step (shared-memory resident pass).
enum TileOpKind : int { TOP_DENSE = 0, TOP_DIAG = 1, TOP_RECIP = 2 };

struct QRef {              // a qubit reference inside a tile: local position or physical bit
    int8_t local;          // tile-local position (>= 0) or -1
    int8_t phys;           // physical bit (used when local < 0)
};

struct Step {
    StepKind kind;
    // ---- Dense / Controlled (streaming, one pass): physical bits
    int k = 0;
    int tpos[5] = {0, 0, 0, 0, 0};
    std::vector<int> ctrl_bits;    // physical
    uint64_t cvals = 0;
    // ---- Diagonal: physical bits of the table index (bit j <- qubit j)
    std::vector<int> dbits;
    // ---- RecipRY
    int anc = 0;
    std::vector<int> clock_bits;   // physical, LSB first
    double delta = 0, snap = 0;
    int is_signed = 1;
    // ---- data (matrix/table) offset into the program's device blob (in double2 units)
    size_t data_off = 0;
    size_t data_len = 0;
    // ---- Tile: sorted physical bits held in shared memory, plus the op list
    std::vector<int> tile_bits;
    std::vector<Gate> tile_ops;    // physical-bit gates (targets/controls are physical bits)
    // register phases of a Tile step: phase p holds ops [phase_start[p], phase_start[p+1]) and
    // keeps the physical bits phase_R[p] (kRegBits of them) in registers
    std::vector<size_t> phase_start;
    std::vector<std::vector<int>> phase_R;
    int reg_bits = 4;              // register bits per phase of this pass (16 or 8 amplitudes per thread)
    // ---- Exchange: swap physical global bits xg[i] with local bits xl[i] (one all-to-all round)
    std::vector<int> xg, xl;
    // ---- InitProduct: factors on physical bits
    std::vector<ProductFactor> factors;
    double bytes = 0;              // HBM bytes this step moves (read + write), per rank
};

struct Program;   // defined in engine.cu (device blob, launch records)

struct CompileOptions {
    int tile_qubits = 12;      // <= 0 : no tiles (one streaming pass per op)
    int wmin = 3;              // tiles always hold the lowest wmin physical bits (128 B segments)
    int reg_bits = 4;          // qubits held in registers per thread in a tile phase (16 amplitudes)
    int jit = 0;               // 0 auto, 1 always, -1 never (NVRTC-specialised tile passes)
    bool reorder = true;       // commutation-aware op reordering for tile packing (single rank)
    int red_qubit = -1;        // >= 0: the last tile pass also accumulates P(logical qubit = 0 / 1) while
                               // it stores the final state (single-rank JIT programs; sv_program::d_mred)
    int diag_merge = 7;        // tile passes: merge consecutive diagonal ops of a register phase into
                               // one table of <= this many qubits after scheduling (0 = off)
    std::vector<int> phys_init;  // programs that start with their own initialisation: logical->physical
                                 // map at program start (empty = identity)
    // host-only planning (hhl_schedule_dump / sv_schedule_dump with tile_jit > 0): program_create
    // lowers and generates every tile pass exactly as for a run, compiles them with NVRTC (no
    // device, no uploads, no launches) and appends one line per launch to *dry_log
    bool dry_run = false;
    std::string *dry_log = nullptr;
    // dry run only: also export the program for host emulation into this directory (blob.bin,
    // launches.txt, src_<i>.cu = generated pass source without the device prelude, cw_<i>.bin)
    std::string emu_dir;
};

// Schedule: logical fused ops (+ optional product init) -> physical steps.
// phys_in: logical->physical map at program start; phys_out: at program end.
struct Schedule {
    std::vector<Step> steps;
    std::vector<int> phys_out;
    uint64_t n_fused = 0;
    double alg_bytes = 0, pass_bytes = 0;
    uint64_t n_passes = 0;
};
Schedule compile(const std::vector<Gate> &ops, const std::vector<ProductFactor> *init, int n, int nloc,
                 const std::vector<int> &phys_in, const CompileOptions &o);
std::string dump_schedule(const Schedule &s);
// SURVEY §8(a) a2 cost model: predicted B200 time (ms) of a schedule of an nloc-qubit (local) state.
double schedule_cost_ms(const Schedule &s, int nloc);

}  // namespace hhlsv
