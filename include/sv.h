/*
 * sv.h — C ABI of the B200-native HHL state-vector hot path (arXiv 2402.08136).
 *
 * The library (paper_2402_08136_b200/libhhlsv.so) simulates the HHL circuit of the
 * paper by full state-vector evolution on sm_100a GPUs: "the most significant time
 * sink is the unitary evolution of the state" (§II-C). Everything on
 * the data path runs in the library's own CUDA kernels; there is NO CPU fallback —
 * without a usable CUDA device every compute entry point returns SV_E_CUDA.
 *
 * Conventions (apply to every call):
 *  - Amplitudes are complex128 stored interleaved (re, im) = CUDA double2.
 *  - Qubit q is bit q of the LOGICAL amplitude index (little-endian; R1).
 *    The library may keep a permuted physical layout internally (qubit relabelling,
 *    global-qubit sharding) but every read/probability/slice is reported in logical
 *    order.
 *  - For a k-qubit matrix, targets[0] is the least-significant bit of its row and
 *    column index; matrices are row-major 2^k × 2^k interleaved complex.
 *  - The caller owns every buffer it passes; the library copies what it needs
 *    (matrices, tables) before the call returns. Objects returned through `out`
 *    pointers are owned by the library until the matching *_destroy call.
 *  - Every call returns sv_status (0 = OK), never throws, never exits;
 *    sv_last_error() gives a thread-local message for the last failure.
 *  - Work is enqueued on the CUDA stream given to sv_create (NULL = legacy default
 *    stream). Calls returning host data synchronise that stream; sv_apply_* and
 *    sv_program_run are asynchronous.
 */
#ifndef HHLSV_SV_H
#define HHLSV_SV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SV_OK = 0,
    SV_E_ARG = 1,          /* bad argument: n < 1, qubit out of range/duplicated, k too large, null ptr, zero b */
    SV_E_RANGE = 2,        /* index range outside the state */
    SV_E_NOTUNITARY = 3,   /* ||U U^† - I||_max > 1e-10 (SPEC S:33 gate invariant) */
    SV_E_NOTHERMITIAN = 4, /* reserved (non-symmetric A is Hermitian-embedded) */
    SV_E_CLOCK = 5,        /* delta = 0: clock register too small for kappa (R5) */
    SV_E_ZEROPROB = 6,     /* post-selection probability < 1e-12 */
    SV_E_OOM = 7,          /* state or workspace does not fit in device memory */
    SV_E_CUDA = 8,         /* CUDA error, or no CUDA device: there is no CPU fallback */
    SV_E_NCCL = 9          /* NCCL error in a multi-GPU exchange/reduction */
} sv_status;

/* Thread-local human-readable message for the last non-OK status on this thread. */
const char *sv_last_error(void);
/* Library version string ("hhlsv <semver> sm_100a"). */
const char *sv_version(void);

/* ------------------------------------------------------------------ state ---- */
typedef struct sv_state sv_state;   /* opaque; library-owned until sv_destroy */

/* Multi-GPU descriptor: one process per GPU. The state of n qubits is
 * sharded by its top log2(world) PHYSICAL qubits; rank r holds the 2^(n-g) amplitudes
 * whose top g physical bits equal r. `nccl_id` points at the 128-byte ncclUniqueId
 * that rank 0 created with sv_nccl_unique_id() and broadcast to all ranks (e.g. with
 * torch.distributed). world must be a power of two. NULL dist = 1 GPU, no NCCL.
 * world > 1 with nccl_id == NULL creates VIRTUAL shards: all `world` shards live in this process
 * on one GPU and global-qubit exchanges are device copies — the same scheduler, rank-resolved
 * kernels and exchange packing as the NCCL path, testable on a single GPU. */
typedef struct {
    int world;
    int rank;
    int device;
    const unsigned char *nccl_id;
} sv_dist;

/* Fill 128 bytes with a fresh ncclUniqueId (rank 0 only). SV_E_NCCL if NCCL cannot be loaded. */
sv_status sv_nccl_unique_id(unsigned char out_id[128]);

/* Transport self-test and microbenchmark of the exchange layer (SURVEY §8(d) "NVLink GB/s per
 * exchange", §5 failure detection): every rank of `world` (one process per GPU, `device`) creates a
 * communicator from the broadcast `nccl_id` and runs `reps` exchanges of the library's own transport
 * (grouped ncclSend/ncclRecv, waited on with the asynchronous-error polling of sharded readouts):
 *   pattern 0 -- pairwise: `bytes` to and from rank ^ 1 (world 1: to itself);
 *   pattern 1 -- all-to-all: bytes / world to and from every other rank (world 1: to itself).
 * Received data are checked against the sender's seeded pattern on the device. Outputs (any may be
 * NULL): ms per exchange (CUDA events on the library stream, median of reps), GB/s = bytes this rank
 * sends per exchange / time, and the number of mismatching doubles (0 = correct). world must be a
 * power of two; bytes a multiple of 8 * world. SV_E_NCCL on a transport failure. */
sv_status sv_comm_bench(int world, int rank, int device, const unsigned char *nccl_id, int pattern, uint64_t bytes,
                        int reps, double *ms_out, double *gbs_out, uint64_t *mismatches_out);

/* Allocate the (local shard of the) state on `dist->device` (or the current device)
 * and initialise it to |0...0>. cuda_stream: a cudaStream_t (NULL = default stream).
 * SV_E_ARG if n_qubits < 1 or n_qubits - log2(world) < 1; SV_E_OOM if it does not fit. */
sv_status sv_create(int n_qubits, const sv_dist *dist, void *cuda_stream, sv_state **out);
sv_status sv_destroy(sv_state *sv);
/* State and workspace memory comes from a stream-ordered pool owned by the library (never the
 * process-wide default pool). Freed memory stays cached for the next state (re-mapping a 16 GiB
 * state costs milliseconds to seconds) and is released when a new state would not fit otherwise, or
 * by this call (device < 0: every device). Synchronises the device. SV_E_CUDA without a device. */
sv_status sv_trim_memory(int device);
/* Re-initialise to |0...0> and reset the logical->physical qubit map to identity. */
sv_status sv_reset(sv_state *sv);
/* Number of qubits / local amplitudes of this rank / the device pointer of the local shard
 * (interleaved double2, PHYSICAL order; valid until sv_destroy). */
sv_status sv_info(sv_state *sv, int *n_qubits, uint64_t *local_amps, void **device_ptr);
/* Current logical->physical qubit map (n ints). */
sv_status sv_qubit_map(sv_state *sv, int *phys_of_logical);
/* Synchronise the library stream. */
sv_status sv_sync(sv_state *sv);

/* Read/write `count` amplitudes starting at LOGICAL index `first` to/from HOST memory
 * (interleaved re,im; 2*count doubles). Multi-GPU: collective — every rank must call it;
 * the values land on every rank. SV_E_RANGE if first+count > 2^n. Synchronous. */
sv_status sv_read(sv_state *sv, uint64_t first, uint64_t count, double *interleaved_out);
sv_status sv_write(sv_state *sv, uint64_t first, uint64_t count, const double *interleaved_in);

/* Checkpoint / restore of the whole state (SPEC "External Interfaces": a uint64 length header then
 * 2^n interleaved re, im doubles, little-endian, LOGICAL order). sv_restore requires the header to
 * equal 2^n of `sv` (SV_E_ARG otherwise, also on I/O errors). Streams through a 64 MiB host buffer.
 * Synchronous; collective when sharded (every rank reads / writes the full logical state). */
sv_status sv_dump(sv_state *sv, const char *path);
sv_status sv_restore(sv_state *sv, const char *path);

/* ------------------------------------------------------------------ gates ---- */
/* Fused-gate IR (SURVEY §2.2 D-FG; the paper's "single fused gate", Fig. 4).
 *  SV_DENSE       targets (1..5): data = 2^k × 2^k matrix.
 *  SV_CONTROLLED  targets (1..5) + controls (1..20) with required values `control_values`
 *                 (bit i = value of controls[i]): data = 2^k × 2^k matrix applied where the
 *                 controls match, identity elsewhere (QPE c-U^(2^j), Fig. 5).
 *  SV_DIAGONAL    targets (1..12): data = 2^k diagonal entries (CP ladders of the (I)QFT).
 *  SV_RECIP_RY    targets[0] = ancilla; controls = the clock register, LSB first (n_c = n_controls);
 *                 data unused. Eigenvalue-inversion rotation (Fig. 5, settings of [qlsarepo],
 *                 PAPER.md:225; R4/R6): for clock value m, L = 2^(n_c - recip_signed),
 *                 m' = m, or 2^n_c - m with sign -1 when recip_signed and m >= 2^(n_c-1);
 *                 r = recip_delta * L / m'; s = 1 if |r-1| <= recip_snap, r if r < 1, else 0
 *                 (s = 0 at m = 0); the ancilla pair gets RY(2 asin(sign*s)).
 *  SV_SWAP        targets = {a, b}: SWAP gate. Executed by relabelling (no data movement).
 */
typedef enum { SV_DENSE = 0, SV_CONTROLLED = 1, SV_DIAGONAL = 2, SV_RECIP_RY = 3, SV_SWAP = 4 } sv_kind;

typedef struct {
    int kind;                  /* sv_kind */
    int n_targets;
    const int *targets;
    int n_controls;
    const int *controls;
    uint64_t control_values;
    const double *data;        /* interleaved complex, see sv_kind */
    double recip_delta;
    int recip_signed;
    double recip_snap;
} sv_gate;

/* Apply gates in order, each as ONE fused operation (no further matrix fusion; the engine
 * may still execute several of them in one HBM pass — DESIGN.md §Passes). Matrices are
 * validated (unitary to 1e-10) and copied. Asynchronous on the library stream. */
sv_status sv_apply_fused(sv_state *sv, const sv_gate *gates, size_t n_gates);

/* Fusion options. fusion_kmax: max dense/controlled target count after
 * fusion (0 = no fusion, 2 = the paper's Fig. 4 mode, 1..5). diag_kmax: max diagonal width
 * (<= 12). tile_qubits: qubits per shared-memory tile pass (0 = library default, -1 =
 * one HBM pass per fused op). */
typedef struct {
    int fusion_kmax;
    int diag_kmax;
    int tile_qubits;
    int tile_jit;       /* 0: auto (NVRTC-specialised tile passes when the local state has >= 2^18 amplitudes),
                           1: always, -1: never (generic interpreting tile kernel) */
    int fusion_mode;    /* 0: structure-preserving greedy window of <= fusion_kmax qubits (default);
                           1: the paper's four prioritised strategies for one-/two-qubit gates (Fig. 4,
                           PAPER.md:207): 1q+1q, 1q into the following 2q, 1q into the preceding 2q, 2q+2q
                           on the same pair (fusion_kmax is ignored) */
} sv_fuse_options;

typedef struct {
    uint64_t n_logical;        /* gates in */
    uint64_t n_fused;          /* fused ops out (excluding swaps, which relabel) */
    uint64_t n_passes;         /* kernel launches over the state the schedule needs */
    double alg_bytes;          /* sum over fused ops of their algorithmic bytes */
    double pass_bytes;         /* HBM bytes the scheduled passes move (read + write) */
} sv_plan_report;

/* Run the a2 fusion pass on a LOGICAL gate list, then apply it (sv_apply_fused semantics). */
sv_status sv_apply_circuit(sv_state *sv, const sv_gate *gates, size_t n_gates, const sv_fuse_options *opt,
                           sv_plan_report *rep);

/* ------------------------------------------------------------- programs ---- */
/* A program is a fused, scheduled gate list resident in device memory (matrices uploaded
 * once), bound to the state it was created for. Running it is stream-ordered and does no
 * host work beyond kernel launches, so it can be timed or captured in a CUDA graph. */
typedef struct sv_program sv_program;
sv_status sv_program_create(sv_state *sv, const sv_gate *gates, size_t n_gates, const sv_fuse_options *opt,
                            sv_program **out, sv_plan_report *rep);
/* Runs the program. A program that starts with a state initialisation (hhl programs) resets
 * the qubit map itself; otherwise the state's qubit map must equal the one at creation. */
sv_status sv_program_run(sv_state *sv, sv_program *prog);
sv_status sv_program_destroy(sv_program *prog);
/* Text dump of the scheduled program (one step per line), for debugging/golden tests. */
sv_status sv_program_dump(sv_program *prog, char *buf, size_t buf_len);
/* Per-launch timing: when enabled, sv_program_run records a CUDA event pair around every
 * kernel launch / exchange on the library stream; sv_program_timings returns the durations
 * (ms) of the last run (synchronises the stream) with each step's kind (0 init-zero,
 * 1 init-product, 2 dense/controlled, 3 diagonal, 4 recip-RY, 5 tile pass, 6 exchange),
 * its HBM bytes per launch, the FP64 flops it must execute (structure-aware: real matrices,
 * butterflies and control-selected amplitudes counted as executed) and how many kernel
 * launches it made. Any output pointer may be NULL. */
sv_status sv_program_set_timing(sv_program *prog, int enable);
sv_status sv_program_timings(sv_program *prog, float *ms, int *kind, double *bytes, double *flops, int *launches,
                             size_t cap, size_t *n_out);
/* Number of kernel launches one sv_program_run makes on this rank, and the host->device
 * bytes uploaded when the program was created. */
sv_status sv_program_stats(sv_program *prog, uint64_t *launches, uint64_t *h2d_bytes);
/* Fused readout (single-GPU HHL programs; SURVEY §8 a8 (ii) for the ancilla, "P(measure
 * ancilla and get 1)"): the program's last tile pass accumulates sum |a|^2 split by the ancilla while it
 * stores the final state, so no separate full-state read is needed. out[0] / out[1] = P(ancilla = 0 / 1)
 * of the last run (their sum is the norm); deterministic (fixed grid, fixed summation order).
 * Synchronises the library stream. SV_E_ARG if the program has no fused marginal (sharded state,
 * no JIT passes, or a program not built by hhl_build_program); use sv_probabilities then. */
sv_status sv_program_marginal(sv_program *prog, double *out2);

/* HOST-ONLY planning (no GPU needed): fuse + schedule a LOGICAL gate list for an n-qubit
 * state sharded over `world` ranks (power of two), and dump the schedule text. Used to test
 * the fusion pass and the global-qubit swap scheduler without a device. */
sv_status sv_schedule_dump(int n_qubits, int world, const sv_gate *gates, size_t n_gates,
                           const sv_fuse_options *opt, char *buf, size_t buf_len, sv_plan_report *rep);

/* --------------------------------------------------------------- readout ---- */
/* Marginal probabilities over LOGICAL `qubits` (bit j of the output index = qubits[j]):
 * out[v] = sum |a_i|^2 over i with bits(i, qubits) = v. out has 2^n_q doubles (n_q <= 26).
 * Deterministic fixed-order reduction (no fp64 atomics). Synchronous; collective when sharded. */
sv_status sv_probabilities(sv_state *sv, const int *qubits, int n_q, double *out);
/* Squared norm sum_i |a_i|^2 (deterministic). Synchronous; collective when sharded. */
sv_status sv_norm2(sv_state *sv, double *out);
/* Post-selection slice ("measure ancilla and get 1", read per DESIGN.md R7):
 * the amplitudes whose LOGICAL qubits fixed_q[i] equal fixed_v[i], in increasing logical
 * order of the remaining qubits. n_out must equal 2^(n - n_fixed) (<= 2^26). amps_out gets
 * 2*n_out doubles, idx_out (optional) the logical indices, prob_out (optional) the summed
 * probability. Synchronous; collective when sharded (results on every rank). */
sv_status sv_postselect_slice(sv_state *sv, const int *fixed_q, const int *fixed_v, int n_fixed,
                              double *amps_out, uint64_t *idx_out, uint64_t n_out, double *prob_out);

/* Shot sampling (SPEC `sample` S:166-174; Fig. 3 caption, "10,000 measurements of the
 * Bell state"): writes `shots` LOGICAL basis indices drawn i.i.d. from |a_i|^2 / sum |a|^2 to out
 * (caller-owned, shots uint64). Deterministic given seed: shot s uses the uniform
 * u_s = (splitmix64(seed + (s+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53 and inverse-CDF search in logical
 * order with the fixed summation order of DESIGN.md §Sampling (the oracle implements the same
 * generator and order, so indices are identical). Single-rank states only (SV_E_ARG when sharded);
 * SV_E_ZEROPROB for a zero state. Synchronous. */
sv_status sv_sample(sv_state *sv, uint64_t shots, uint64_t seed, uint64_t *out);

/* ------------------------------------------------------------------- HHL ---- */
/* HHL front end + solve ("Practical HHL procedures", Fig. 5, resources
 * PAPER.md:225-242 read per DESIGN.md R2/R3). */
typedef struct {
    int clock_qubits;   /* n_c including the sign qubit; <= 0: max(n_b+1, ceil(log2(kappa+1))) + 1 */
    int fusion_kmax;    /* 0 -> chosen by the a2 cost model among 1..5 (predicted time of each
                           candidate schedule from HBM bytes, FP64 flops, register-phase exchanges,
                           launches, NVLink exchanges); -1 -> no fusion; 1..5 -> that width */
    int tile_qubits;    /* 0 -> library default ; -1 -> one pass per fused op */
    double recip_snap;  /* reciprocal snapping tolerance (qlsarepo: 1e-5); < 0 -> default 1e-5 */
    int init_fold;      /* 0 (default): fold the leading product-state gates into the init kernel; 1: also the
                           diagonal gates right after them; -1: no folding */
    int tile_jit;       /* as sv_fuse_options.tile_jit */
    int diag_kmax;      /* max qubits of a diagonal fused BEFORE scheduling (0 -> 4 with tile passes: the tile
                           scheduler places small diagonals freely and merges those of one register phase
                           into <= 8-qubit tables afterwards; 12 without tile passes) */
    int qpe_mode;       /* 0: textbook circuit (c-U^(2^j) blocks, Fig. 5); 1: eigenbasis rewrite:
                           c-U_j = V diag(e^{2 pi i frac(2^j phi_s)}) V^T, so the controlled chain becomes
                           V^T, one diagonal phase factor per clock bit over (system, clock bit), V — the
                           same unitary (parity is checked against the textbook oracle) */
    /* Optional caller-supplied eigendecomposition of the PADDED (and, for a non-symmetric A,
     * Hermitian-embedded) N_p x N_p system matrix (N_p = 2^n_data), used instead of the library's
     * Jacobi eigensolver (step 2 of PAPER.md:156-199): eig_lambda[s] (N_p doubles) and eig_vectors
     * (N_p x N_p, row-major, column s = unit eigenvector of eig_lambda[s]: the numpy.linalg.eigh
     * layout). Both NULL (default) -> the library computes them. Checked: SV_E_ARG when
     * max|A v_s - lambda_s v_s| > 1e-8 max(1, max|lambda|) or V is not orthogonal to 1e-10.
     * Use: reproducing another eigensolver's phases bit for bit (the HHL state is sensitive to
     * phi_s with gain ~2 pi 2^n_c). */
    const double *eig_lambda;
    const double *eig_vectors;
    int fusion_mode;    /* as sv_fuse_options.fusion_mode */
    int fused_marginal; /* hhl_build_program: 1 -> the program's last tile pass also accumulates P(ancilla) while
                           it stores the final state (sv_program_marginal; single GPU, NVRTC passes; costs
                           ~1 % of the run); 0 (default) -> not. hhl_solve always fuses it when it can (it
                           replaces the separate full-state read of the readout). */
} hhl_options;

typedef struct {
    double p_success;   /* P(ancilla = 1 and clock = 0) (R7) */
    double norm2;       /* ||psi||^2 after the circuit (should be 1) */
    double lambda_min, lambda_max, kappa, delta, t_evol;
    int n_data, n_clock, n_total;
    uint64_t n_logical, n_fused, n_passes;
    double alg_bytes, pass_bytes;
    double t_frontend_s, t_sim_s;
    double h2d_bytes, d2h_bytes;   /* host<->device bytes of one solve (program upload, slice read) */
    int x_offset;                  /* Hermitian embedding of a non-symmetric A: x = lower half of the slice */
    int n_orig;                    /* N of the caller's system (before padding / embedding) */
    double b_norm;                 /* ||b||_2 of the caller's b (set by hhl_build_program / hhl_solve):
                                      the scale of step 4's recovery, PAPER.md:193-198 */
    double p_anc1;                 /* P(ancilla = 1) summed over every clock value (hhl_solve only;
                                      the paper's "measure ancilla and get 1", before
                                      the clock = 0 post-selection of R7) */
    int fusion_kmax_used;          /* fusion width used (the cost model's choice when fusion_kmax = 0) */
    double model_ms;               /* the a2 cost model's predicted B200 time of the schedule (ms) */
} hhl_report;

/* hhl_plan_size: the register sizes (n_data, n_clock, n_total) hhl_build_program needs for (A, b).
 * hhl_build_program: build the HHL circuit for A (N×N, row-major, real; a non-symmetric A is embedded
 * as [[0, A], [A^T, 0]] [0; x] = [b; 0]) and b (N) and return it as a program for
 * `sv` (which must have n_total qubits). rep (optional) receives the plan (lambda_min, b_norm, sizes,
 * schedule figures): it is what hhl_readout needs. */
sv_status hhl_plan_size(const double *A, const double *b, int N, const hhl_options *opt, int *n_data,
                        int *n_clock, int *n_total);
sv_status hhl_build_program(sv_state *sv, const double *A, const double *b, int N, const hhl_options *opt,
                            sv_program **out, hhl_report *rep);
/* HOST-ONLY (no GPU needed): plan, build, fold and fuse the HHL circuit for (A, b) exactly as
 * hhl_build_program does, schedule it for `world` ranks (power of two) and write the schedule
 * text (one line per step, ops indented) into buf (NUL-terminated, truncated to buf_len).
 * rep (may be NULL) receives the plan and schedule sizes; its timing fields are zero. */
sv_status hhl_schedule_dump(const double *A, const double *b, int N, const hhl_options *opt, int world, char *buf,
                            size_t buf_len, hhl_report *rep);
/* Read out and recover x after the program ran (PAPER.md:193-198 step 4, read per F3/R8):
 * post-select ancilla = 1, clock = 0 (R7), P = the slice's squared norm, |x> = slice / sqrt(P),
 * x = rep->b_norm * sqrt(P) / rep->lambda_min * |x> (real part, padding / embedding stripped).
 * rep = the report hhl_build_program filled. x_out has N doubles; N must equal rep->n_orig
 * (SV_E_ARG otherwise). SV_E_ZEROPROB when P < 1e-12. p_success (optional) receives P. */
sv_status hhl_readout(sv_state *sv, const hhl_report *rep, int N, double *x_out, double *p_success);
/* Everything at once: create the state, build, run, read out, recover, destroy.
 * A, b, x_out are HOST buffers. dist = NULL for 1 GPU. */
sv_status hhl_solve(const double *A, const double *b, int N, int clock_qubits, const hhl_options *opt,
                    const sv_dist *dist, void *cuda_stream, double *x_out, hhl_report *rep);

#ifdef __cplusplus
}
#endif
#endif /* HHLSV_SV_H */
