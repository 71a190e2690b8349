// The extern "C" boundary declared in include/sv.h. Argument marshalling and error
// translation only; all data-path work happens in the CUDA kernels behind engine.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <new>

#include "comm.h"
#include "engine.h"

using namespace hhlsv;

namespace {
thread_local std::string g_last_error;

template <class F>
sv_status guard(F &&f) {
    try {
        f();
        return SV_OK;
    } catch (const Error &e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc &) {
        g_last_error = "host out of memory";
        return SV_E_OOM;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return SV_E_ARG;
    }
}

std::vector<Gate> gates_in_n(int nq, const sv_gate *g, size_t n) {
    if (n && !g) fail(SV_E_ARG, "null gate array");
    std::vector<Gate> out;
    out.reserve(n);
    for (size_t i = 0; i < n; i++) out.push_back(gate_from_abi(g[i], nq));
    return out;
}

std::vector<Gate> gates_in(const sv_state *sv, const sv_gate *g, size_t n) { return gates_in_n(sv->n, g, n); }

FuseOptions fuse_opts(const sv_fuse_options *o) {
    FuseOptions f;
    if (o) {
        f.kmax = o->fusion_kmax;
        if (o->diag_kmax > 0) f.diag_kmax = o->diag_kmax;
        if (o->fusion_mode < 0 || o->fusion_mode > 1) fail(SV_E_ARG, "fusion_mode must be 0 or 1");
        f.mode = o->fusion_mode;
    }
    if (f.kmax > 5) fail(SV_E_ARG, "fusion_kmax must be <= 5");
    if (f.diag_kmax > 12) fail(SV_E_ARG, "diag_kmax must be <= 12");
    return f;
}

CompileOptions compile_opts(const sv_fuse_options *o) {
    CompileOptions c;
    if (o && o->tile_qubits != 0) c.tile_qubits = o->tile_qubits;
    if (o) c.jit = o->tile_jit;
    return c;
}

void fill_plan_report(const sv_program *p, sv_plan_report *rep) {
    if (!rep) return;
    rep->n_logical = p->n_logical;
    rep->n_fused = p->sched.n_fused;
    rep->n_passes = p->sched.n_passes;
    rep->alg_bytes = p->sched.alg_bytes;
    rep->pass_bytes = p->sched.pass_bytes;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

const char *sv_last_error(void) { return g_last_error.c_str(); }
const char *sv_version(void) { return "hhlsv 0.1.0 sm_100a"; }

sv_status sv_nccl_unique_id(unsigned char out_id[128]) {
    return guard([&] {
        if (!out_id) fail(SV_E_ARG, "null id buffer");
        if (nccl_unique_id(out_id)) fail(SV_E_NCCL, std::string("ncclGetUniqueId: ") + nccl_last_error());
    });
}

sv_status sv_comm_bench(int world, int rank, int device, const unsigned char *nccl_id, int pattern, uint64_t bytes,
                        int reps, double *ms_out, double *gbs_out, uint64_t *mismatches_out) {
    return guard([&] {
        if (!nccl_id) fail(SV_E_ARG, "null nccl_id");
        if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world)
            fail(SV_E_ARG, "world must be a power of two and 0 <= rank < world");
        if (pattern != 0 && pattern != 1) fail(SV_E_ARG, "pattern must be 0 (pairwise) or 1 (all-to-all)");
        if (reps < 1 || bytes == 0 || bytes % (8ull * (uint64_t)world))
            fail(SV_E_ARG, "reps >= 1 and bytes a positive multiple of 8 * world");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
            cudaGetLastError();
            fail(SV_E_CUDA, "no CUDA device: this library has no CPU fallback");
        }
        if (device >= 0) cuda_check(cudaSetDevice(device), "cudaSetDevice");
        struct Res {              // released on every exit path
            Comm c;
            cudaStream_t s = nullptr;
            double *sb = nullptr, *rb = nullptr;
            unsigned long long *bad = nullptr;
            cudaEvent_t e[2] = {nullptr, nullptr};
            ~Res() {
                if (s) cudaStreamSynchronize(s);
                cudaFree(sb);
                cudaFree(rb);
                cudaFree(bad);
                for (auto ev : e)
                    if (ev) cudaEventDestroy(ev);
                if (s) cudaStreamDestroy(s);
                nccl_destroy(c);
            }
        } r;
        if (nccl_init(r.c, world, rank, nccl_id)) fail(SV_E_NCCL, std::string("ncclCommInitRank: ") + nccl_last_error());
        cuda_check(cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking), "stream");
        const uint64_t n = bytes / 8;
        cuda_check(cudaMalloc((void **)&r.sb, bytes), "cudaMalloc(send)");
        cuda_check(cudaMalloc((void **)&r.rb, bytes), "cudaMalloc(recv)");
        cuda_check(cudaMalloc((void **)&r.bad, sizeof(unsigned long long)), "cudaMalloc(count)");
        cuda_check(cudaMemsetAsync(r.bad, 0, sizeof(unsigned long long), r.s), "memset");
        cuda_check(cudaMemsetAsync(r.rb, 0xff, bytes, r.s), "memset");       // NaN until received
        cuda_check(dev::launch_fill_pattern(r.sb, n, (uint64_t)rank, 0, r.s), "fill");
        // (peer, chunk): pairwise -> the whole buffer with rank ^ 1; all-to-all -> chunk p with rank p
        std::vector<int> peers;
        std::vector<const double *> sp;
        std::vector<double *> rp;
        std::vector<uint64_t> roff;       // offset of the received chunk in the sender's pattern
        uint64_t cnt = n;
        if (pattern == 0) {
            const int peer = world == 1 ? 0 : (rank ^ 1);
            peers = {peer};
            sp = {r.sb};
            rp = {r.rb};
            roff = {0};
        } else {
            cnt = n / (uint64_t)world;
            for (int q = 0; q < world; q++) {
                if (world > 1 && q == rank) continue;
                peers.push_back(q);
                sp.push_back(r.sb + (uint64_t)q * cnt);
                rp.push_back(r.rb + (uint64_t)q * cnt);
                roff.push_back((uint64_t)rank * cnt);
            }
        }
        for (auto &ev : r.e) cuda_check(cudaEventCreate(&ev), "event");
        std::vector<float> ms;
        for (int i = 0; i < reps + 1; i++) {          // one untimed warm-up exchange
            cuda_check(cudaEventRecord(r.e[0], r.s), "event");
            if (nccl_alltoall_pairs(r.c, sp.data(), rp.data(), peers.data(), (int)peers.size(), cnt, r.s))
                fail(SV_E_NCCL, std::string("exchange: ") + nccl_last_error());
            cuda_check(cudaEventRecord(r.e[1], r.s), "event");
            if (nccl_wait(r.c, r.s, 300.0)) fail(SV_E_NCCL, std::string("exchange wait: ") + nccl_last_error());
            float t = 0.0f;
            cuda_check(cudaEventElapsedTime(&t, r.e[0], r.e[1]), "elapsed");
            if (i) ms.push_back(t);
        }
        for (size_t i = 0; i < peers.size(); i++)
            cuda_check(dev::launch_check_pattern(rp[i], cnt, (uint64_t)peers[i], roff[i], r.bad, r.s), "check");
        unsigned long long bad = 0;
        cuda_check(cudaMemcpyAsync(&bad, r.bad, sizeof bad, cudaMemcpyDeviceToHost, r.s), "count d2h");
        cuda_check(cudaStreamSynchronize(r.s), "sync");
        std::sort(ms.begin(), ms.end());
        const double med = ms[ms.size() / 2];
        const double sent = 8.0 * (double)cnt * (double)peers.size();
        if (ms_out) *ms_out = med;
        if (gbs_out) *gbs_out = med > 0 ? sent / (med * 1e-3) / 1e9 : 0.0;
        if (mismatches_out) *mismatches_out = bad;
    });
}

sv_status sv_create(int n_qubits, const sv_dist *dist, void *cuda_stream, sv_state **out) {
    return guard([&] {
        if (!out) fail(SV_E_ARG, "null out");
        *out = nullptr;
        *out = state_create(n_qubits, dist, (cudaStream_t)cuda_stream);
    });
}

sv_status sv_destroy(sv_state *sv) {
    return guard([&] { state_destroy(sv); });
}

sv_status sv_trim_memory(int device) {
    return guard([&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
            cudaGetLastError();
            fail(SV_E_CUDA, "no CUDA device: this library has no CPU fallback");
        }
        cuda_check(cudaDeviceSynchronize(), "sync before trim");
        pool_trim(device, 0);
    });
}

sv_status sv_reset(sv_state *sv) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        state_reset(sv);
    });
}

sv_status sv_info(sv_state *sv, int *n, uint64_t *local_amps, void **ptr) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        if (n) *n = sv->n;
        if (local_amps) *local_amps = sv->local_amps();
        if (ptr) *ptr = sv->psi;
    });
}

sv_status sv_qubit_map(sv_state *sv, int *phys) {
    return guard([&] {
        if (!sv || !phys) fail(SV_E_ARG, "null argument");
        for (int q = 0; q < sv->n; q++) phys[q] = sv->phys[q];
    });
}

sv_status sv_sync(sv_state *sv) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        cuda_check(cudaStreamSynchronize(sv->stream), "sync");
    });
}

sv_status sv_read(sv_state *sv, uint64_t first, uint64_t count, double *out) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        state_read(sv, first, count, out);
    });
}

sv_status sv_write(sv_state *sv, uint64_t first, uint64_t count, const double *in) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        state_write(sv, first, count, in);
    });
}

// State dump / restore (SPEC "External Interfaces": length header + interleaved re/im doubles, little-
// endian), in LOGICAL order, streamed through a bounded host buffer. Collective when sharded: every rank
// reads / writes the whole logical state (rank 0's file is the one to keep).
static const uint64_t kDumpChunk = 1ull << 22;     // amplitudes per chunk (64 MiB of host buffer)

sv_status sv_dump(sv_state *sv, const char *path) {
    return guard([&] {
        if (!sv || !path) fail(SV_E_ARG, "null argument");
        FILE *f = fopen(path, "wb");
        if (!f) fail(SV_E_ARG, std::string("cannot open ") + path);
        const uint64_t N = 1ull << sv->n;
        std::vector<double> buf(2 * std::min(N, kDumpChunk));
        bool ok = fwrite(&N, sizeof N, 1, f) == 1;
        for (uint64_t off = 0; ok && off < N; off += kDumpChunk) {
            const uint64_t c = std::min(kDumpChunk, N - off);
            try {
                state_read(sv, off, c, buf.data());
            } catch (...) {
                fclose(f);
                throw;
            }
            ok = fwrite(buf.data(), sizeof(double), 2 * c, f) == 2 * c;
        }
        if (fclose(f) != 0 || !ok) fail(SV_E_ARG, std::string("write failed: ") + path);
    });
}

sv_status sv_restore(sv_state *sv, const char *path) {
    return guard([&] {
        if (!sv || !path) fail(SV_E_ARG, "null argument");
        FILE *f = fopen(path, "rb");
        if (!f) fail(SV_E_ARG, std::string("cannot open ") + path);
        uint64_t N = 0;
        const uint64_t want = 1ull << sv->n;
        if (fread(&N, sizeof N, 1, f) != 1 || N != want) {
            fclose(f);
            fail(SV_E_ARG, "dump header does not match the state size");
        }
        std::vector<double> buf(2 * std::min(N, kDumpChunk));
        for (uint64_t off = 0; off < N; off += kDumpChunk) {
            const uint64_t c = std::min(kDumpChunk, N - off);
            if (fread(buf.data(), sizeof(double), 2 * c, f) != 2 * c) {
                fclose(f);
                fail(SV_E_ARG, "dump truncated");
            }
            try {
                state_write(sv, off, c, buf.data());
            } catch (...) {
                fclose(f);
                throw;
            }
        }
        fclose(f);
    });
}

sv_status sv_apply_fused(sv_state *sv, const sv_gate *gates, size_t n_gates) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        auto g = gates_in(sv, gates, n_gates);
        sv_program *p = program_create(sv, g, nullptr, CompileOptions{}, n_gates);
        try {
            program_run(sv, p);
        } catch (...) {
            program_destroy(p);
            throw;
        }
        program_destroy(p);
    });
}

sv_status sv_apply_circuit(sv_state *sv, const sv_gate *gates, size_t n_gates, const sv_fuse_options *opt,
                           sv_plan_report *rep) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        auto g = fuse(gates_in(sv, gates, n_gates), fuse_opts(opt));
        sv_program *p = program_create(sv, g, nullptr, compile_opts(opt), n_gates);
        fill_plan_report(p, rep);
        try {
            program_run(sv, p);
        } catch (...) {
            program_destroy(p);
            throw;
        }
        program_destroy(p);
    });
}

sv_status sv_program_create(sv_state *sv, const sv_gate *gates, size_t n_gates, const sv_fuse_options *opt,
                            sv_program **out, sv_plan_report *rep) {
    return guard([&] {
        if (!sv || !out) fail(SV_E_ARG, "null argument");
        *out = nullptr;
        auto g = fuse(gates_in(sv, gates, n_gates), fuse_opts(opt));
        *out = program_create(sv, g, nullptr, compile_opts(opt), n_gates);
        fill_plan_report(*out, rep);
    });
}

sv_status sv_program_run(sv_state *sv, sv_program *prog) {
    return guard([&] {
        if (!sv || !prog) fail(SV_E_ARG, "null argument");
        program_run(sv, prog);
    });
}

sv_status sv_program_destroy(sv_program *prog) {
    return guard([&] { program_destroy(prog); });
}

sv_status sv_program_dump(sv_program *prog, char *buf, size_t len) {
    return guard([&] {
        if (!prog || !buf || len == 0) fail(SV_E_ARG, "null argument");
        std::string s = dump_schedule(prog->sched);
        size_t n = std::min(len - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    });
}

sv_status sv_program_set_timing(sv_program *prog, int enable) {
    return guard([&] {
        if (!prog) fail(SV_E_ARG, "null program");
        prog->timing = enable != 0;
    });
}

sv_status sv_program_timings(sv_program *prog, float *ms, int *kind, double *bytes, double *flops, int *launches,
                             size_t cap, size_t *n_out) {
    return guard([&] {
        if (!prog) fail(SV_E_ARG, "null program");
        program_timings(prog, ms, kind, bytes, flops, launches, cap, n_out);
    });
}

sv_status sv_program_stats(sv_program *prog, uint64_t *launches, uint64_t *h2d_bytes) {
    return guard([&] {
        if (!prog) fail(SV_E_ARG, "null program");
        if (launches) *launches = prog->launches();
        if (h2d_bytes) *h2d_bytes = (uint64_t)prog->h2d_bytes;
    });
}

sv_status sv_program_marginal(sv_program *prog, double *out2) {
    return guard([&] {
        if (!prog || !out2) fail(SV_E_ARG, "null argument");
        if (!prog->d_mred) fail(SV_E_ARG, "program has no fused marginal");
        cuda_check(cudaMemcpyAsync(out2, prog->d_mred + 2 * sv_program::kMredCtas, 2 * sizeof(double),
                                   cudaMemcpyDeviceToHost, prog->sv->stream),
                   "marginal d2h");
        cuda_check(cudaStreamSynchronize(prog->sv->stream), "marginal sync");
    });
}

// Host-only: generate + NVRTC-compile every tile pass of a schedule; one log line per pass.
sv_status sv_schedule_dump(int n_qubits, int world, const sv_gate *gates, size_t n_gates, const sv_fuse_options *opt,
                           char *buf, size_t buf_len, sv_plan_report *rep) {
    return guard([&] {
        if (world < 1 || (world & (world - 1))) fail(SV_E_ARG, "world must be a power of two");
        int g = 0;
        while ((1 << g) < world) g++;
        if (n_qubits < 1 || n_qubits - g < 1 || n_qubits > 62) fail(SV_E_ARG, "n_qubits out of range");
        auto gl = fuse(gates_in_n(n_qubits, gates, n_gates), fuse_opts(opt));
        std::vector<int> phys(n_qubits);
        for (int q = 0; q < n_qubits; q++) phys[q] = q;
        CompileOptions co = compile_opts(opt);
        if (co.tile_qubits > 14) co.tile_qubits = 14;
        std::string jitlog;
        Schedule s;
        if (opt && opt->tile_jit > 0) {     // rank 0's program exactly as sv_program_create lowers it (host only)
            sv_state host{};
            host.n = n_qubits;
            host.g = g;
            host.nloc = n_qubits - g;
            host.world = world;
            host.phys = phys;
            co.dry_run = true;
            co.dry_log = &jitlog;
            if (const char *e = getenv("HHLSV_EMU_DIR")) co.emu_dir = e;     // test tooling (tests/jit_emulator.py)
            std::unique_ptr<sv_program> prog(program_create(&host, gl, nullptr, co, n_gates));
            s = prog->sched;
        } else {
            s = compile(gl, nullptr, n_qubits, n_qubits - g, phys, co);
        }
        if (rep) {
            rep->n_logical = n_gates;
            rep->n_fused = s.n_fused;
            rep->n_passes = s.n_passes;
            rep->alg_bytes = s.alg_bytes;
            rep->pass_bytes = s.pass_bytes;
        }
        if (buf && buf_len) {
            std::string t = dump_schedule(s) + jitlog;
            std::string perm = "FINAL_MAP";
            for (int q = 0; q < n_qubits; q++) perm += " " + std::to_string(s.phys_out[q]);
            t += perm + "\n";
            size_t n = std::min(buf_len - 1, t.size());
            std::memcpy(buf, t.data(), n);
            buf[n] = 0;
        }
    });
}

sv_status sv_probabilities(sv_state *sv, const int *qubits, int n_q, double *out) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        state_probabilities(sv, qubits, n_q, out);
    });
}

sv_status sv_norm2(sv_state *sv, double *out) {
    return guard([&] {
        if (!sv || !out) fail(SV_E_ARG, "null argument");
        *out = state_norm2(sv);
    });
}

sv_status sv_postselect_slice(sv_state *sv, const int *fixed_q, const int *fixed_v, int n_fixed, double *amps_out,
                              uint64_t *idx_out, uint64_t n_out, double *prob_out) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        state_postselect(sv, fixed_q, fixed_v, n_fixed, amps_out, idx_out, n_out, prob_out);
    });
}

sv_status sv_sample(sv_state *sv, uint64_t shots, uint64_t seed, uint64_t *out) {
    return guard([&] {
        if (!sv) fail(SV_E_ARG, "null state");
        state_sample(sv, shots, seed, out);
    });
}

// ------------------------------------------------------------------- HHL ----
static double opt_snap(const hhl_options *o) { return (o && o->recip_snap >= 0.0) ? o->recip_snap : 1e-5; }
static HHLPlanHost plan_of(const double *A, const double *b, int N, const hhl_options *o) {
    return hhl_plan(A, b, N, o ? o->clock_qubits : 0, opt_snap(o), o ? o->eig_lambda : nullptr,
                    o ? o->eig_vectors : nullptr);
}
// the plan fields of hhl_report (sizes, spectrum, delta/t, b_norm)
static void report_plan(hhl_report *rep, const HHLPlanHost &p) {
    std::memset(rep, 0, sizeof(*rep));
    rep->lambda_min = p.lam_min;
    rep->lambda_max = p.lam_max;
    rep->kappa = p.kappa;
    rep->delta = p.delta;
    rep->t_evol = p.t;
    rep->n_data = p.n_b;
    rep->n_clock = p.n_c;
    rep->n_total = p.n;
    rep->x_offset = p.x_offset;
    rep->n_orig = p.n_orig;
    rep->b_norm = p.b_norm;
}

sv_status hhl_plan_size(const double *A, const double *b, int N, const hhl_options *opt, int *n_data, int *n_clock,
                        int *n_total) {
    return guard([&] {
        HHLPlanHost p = plan_of(A, b, N, opt);
        if (n_data) *n_data = p.n_b;
        if (n_clock) *n_clock = p.n_c;
        if (n_total) *n_total = p.n;
    });
}

// Host part of the HHL program: logical circuit, product-state prefix folded into init factors,
// fusion of the rest. Shared by hhl_build_program and the host-only hhl_schedule_dump.
struct FuseChoice {
    int kmax = 0;                 // fusion width used
    double model_ms = 0.0;        // cost-model prediction of the chosen schedule
};

// Host part of the HHL program: logical circuit, product-state prefix folded into init factors,
// fusion of the rest. fusion_kmax = 0 (default): the a2 cost model (compile.cpp schedule_cost_ms)
// picks the width among 1..5 by scheduling each candidate for this state (nloc local qubits, initial
// layout phys) and predicting its B200 time. Shared by hhl_build_program and hhl_schedule_dump.
static std::vector<Gate> hhl_fused_gates(const HHLPlanHost &p, const hhl_options *opt,
                                         std::vector<ProductFactor> &factors, size_t *n_logical,
                                         const CompileOptions &co, int nloc, FuseChoice *choice) {
    std::vector<Gate> gates = hhl_build(p, opt ? opt->qpe_mode : 0);
    prof_mark("hhl_build");
    const bool fold = !opt || opt->init_fold >= 0;
    size_t nf = fold ? fold_product_prefix(gates, p.n, factors, opt && opt->init_fold == 1) : 0;
    std::vector<Gate> rest(gates.begin() + nf, gates.end());
    FuseOptions fo;
    if (opt && opt->fusion_kmax != 0) fo.kmax = opt->fusion_kmax < 0 ? 0 : opt->fusion_kmax;
    if (fo.kmax > 5) fail(SV_E_ARG, "fusion_kmax must be <= 5");
    // tile passes: keep diagonals small before scheduling (placed freely, merged per register phase
    // afterwards); one HBM pass per op: merge them up front
    fo.diag_kmax = (opt && opt->tile_qubits < 0) ? 12 : 4;
    if (opt && opt->diag_kmax > 0) fo.diag_kmax = std::min(12, opt->diag_kmax);
    if (opt && (opt->fusion_mode < 0 || opt->fusion_mode > 1)) fail(SV_E_ARG, "fusion_mode must be 0 or 1");
    if (opt) fo.mode = opt->fusion_mode;
    if (n_logical) *n_logical = gates.size();
    std::vector<int> phys(p.n);
    for (int q = 0; q < p.n; q++) phys[q] = q;
    if (!co.phys_init.empty()) phys = co.phys_init;
    CompileOptions cc = co;
    if (cc.tile_qubits > 12) cc.tile_qubits = 12;
    const bool auto_k = (!opt || opt->fusion_kmax == 0) && fo.mode == 0;
    if (!auto_k) {
        std::vector<Gate> f = fuse(rest, fo);
        if (choice) {       // model time of the fixed width: from the schedule the caller compiles anyway
            choice->kmax = fo.kmax;
            choice->model_ms = NAN;
        }
        return f;
    }
    std::vector<Gate> best;
    double best_ms = INFINITY;
    int best_k = 1;
    for (int k = 1; k <= 5; k++) {
        FuseOptions fk = fo;
        fk.kmax = k;
        std::vector<Gate> f = fuse(rest, fk);
        const double ms = schedule_cost_ms(compile(f, factors.empty() ? nullptr : &factors, p.n, nloc, phys, cc), nloc);
        if (ms < best_ms * (1.0 - 1e-9)) {      // ties: the narrower width
            best_ms = ms;
            best_k = k;
            best = std::move(f);
        }
    }
    prof_mark("fusion width (cost model)");
    if (choice) {
        choice->kmax = best_k;
        choice->model_ms = best_ms;
    }
    return best;
}

// Initial physical layout of a SHARDED eigenbasis HHL program, g global
// qubits: the top g SYSTEM qubits take the global bits and [system rest | clock | ancilla] the local
// ones. In the eigenbasis circuit the system register is touched non-diagonally only by V^T (folded
// into the product init, which is rank-resolved) and by the final V, so every Hadamard of the
// (I)QFT / H layers, the reciprocal rotation and all diagonal phase tables (rank-resolved table
// slices) run without communication; the final V needs ONE exchange round, whose victims (clock /
// ancilla qubits whose last use is past, chosen by the scheduler) never return. Single rank, the
// textbook circuit or g > n_b: identity (the top logical qubits -- ancilla, clock MSBs -- global).
static std::vector<int> hhl_layout(const HHLPlanHost &p, const hhl_options *opt, int g) {
    if (g < 1 || !opt || opt->qpe_mode != 1 || g > p.n_b) return {};
    std::vector<int> phys(p.n, -1);
    int next = 0;
    for (int s = 0; s < p.n_b - g; s++) phys[s] = next++;          // local system qubits
    for (int j = 0; j < p.n_c; j++) phys[p.n_b + j] = next++;       // clock register
    phys[p.n - 1] = next++;                                        // ancilla
    for (int s = p.n_b - g; s < p.n_b; s++) phys[s] = next++;      // global: top system qubits
    return phys;
}

static CompileOptions hhl_compile_opts(const hhl_options *opt, const HHLPlanHost *p = nullptr, int g = 0,
                                       bool marginal = false) {
    CompileOptions co;
    if (opt && opt->tile_qubits != 0) co.tile_qubits = opt->tile_qubits;
    if (opt) co.jit = opt->tile_jit;
    if (p) co.phys_init = hhl_layout(*p, opt, g);
    // single-GPU programs: the last tile pass also accumulates P(ancilla) (hhl_report.p_anc1, norm2)
    if (p && g == 0 && (marginal || (opt && opt->fused_marginal))) co.red_qubit = p->n - 1;
    return co;
}

static sv_program *build_hhl(sv_state *sv, const HHLPlanHost &p, const hhl_options *opt, hhl_report *rep,
                             double t0, bool marginal = false) {
    prof_mark("build_hhl start");
    if (p.n != sv->n) fail(SV_E_ARG, "state has the wrong number of qubits for this system (use hhl_plan_size)");
    std::vector<ProductFactor> factors;
    size_t n_logical = 0;
    const CompileOptions hco = hhl_compile_opts(opt, &p, sv->n - sv->nloc, marginal);
    FuseChoice fc;
    std::vector<Gate> fused = hhl_fused_gates(p, opt, factors, &n_logical, hco, sv->nloc, &fc);
    prof_mark("fold + fuse");
    sv_program *prog = program_create(sv, fused, &factors, hco, n_logical);
    prof_mark("program_create");
    if (rep) {
        report_plan(rep, p);
        rep->n_logical = n_logical;
        rep->n_fused = prog->sched.n_fused;
        rep->n_passes = prog->sched.n_passes;
        rep->alg_bytes = prog->sched.alg_bytes;
        rep->pass_bytes = prog->sched.pass_bytes;
        rep->h2d_bytes = prog->h2d_bytes;
        rep->d2h_bytes = 16.0 * (double)(1ull << p.n_b) + 8.0;
        rep->fusion_kmax_used = fc.kmax;
        rep->model_ms = std::isnan(fc.model_ms) ? schedule_cost_ms(prog->sched, sv->nloc) : fc.model_ms;
        rep->t_frontend_s = now_s() - t0;
    }
    return prog;
}

sv_status hhl_build_program(sv_state *sv, const double *A, const double *b, int N, const hhl_options *opt,
                            sv_program **out, hhl_report *rep) {
    return guard([&] {
        if (!sv || !out) fail(SV_E_ARG, "null argument");
        *out = nullptr;
        const double t0 = now_s();
        *out = build_hhl(sv, plan_of(A, b, N, opt), opt, rep, t0);
    });
}

static void readout(sv_state *sv, const hhl_report *rep, int N, double *x_out, double *p_out) {
    const int nb = rep->n_data, nc = rep->n_clock, n = rep->n_total;
    if (n != sv->n || nb < 1 || nc < 1 || nb + nc + 1 != n) fail(SV_E_ARG, "report does not match the state");
    if (N != rep->n_orig || N < 1 || rep->x_offset < 0 || (uint64_t)rep->x_offset + (uint64_t)N > (1ull << nb))
        fail(SV_E_ARG, "N does not match the report (N must equal rep->n_orig)");
    if (!(rep->lambda_min > 0.0) || !(rep->b_norm > 0.0)) fail(SV_E_ARG, "report lacks lambda_min / b_norm");
    std::vector<int> fq, fv;
    for (int j = 0; j < nc; j++) {
        fq.push_back(nb + j);
        fv.push_back(0);
    }
    fq.push_back(n - 1);
    fv.push_back(1);
    const uint64_t m = 1ull << nb;
    std::vector<double> amps(2 * m);
    double P = 0.0;
    state_postselect(sv, fq.data(), fv.data(), (int)fq.size(), amps.data(), nullptr, m, &P);
    if (p_out) *p_out = P;
    if (P < 1e-12) fail(SV_E_ZEROPROB, "post-selection probability below 1e-12");
    // x = ||b|| sqrt(P)/lambda_min * slice/sqrt(P)   (PAPER.md:193-198 read per F3/R8)
    if (x_out)
        for (int i = 0; i < N; i++) x_out[i] = rep->b_norm * amps[2 * (rep->x_offset + i)] / rep->lambda_min;
}

sv_status hhl_schedule_dump(const double *A, const double *b, int N, const hhl_options *opt, int world, char *buf,
                            size_t buf_len, hhl_report *rep) {
    return guard([&] {
        if (world < 1 || (world & (world - 1))) fail(SV_E_ARG, "world must be a power of two");
        int g = 0;
        while ((1 << g) < world) g++;
        HHLPlanHost p = plan_of(A, b, N, opt);
        if (p.n - g < 1) fail(SV_E_ARG, "too many ranks for this system");
        std::vector<ProductFactor> factors;
        size_t n_logical = 0;
        FuseChoice fc;
        std::vector<Gate> fused = hhl_fused_gates(p, opt, factors, &n_logical, hhl_compile_opts(opt, &p, g), p.n - g, &fc);
        // rank 0's program exactly as hhl_build_program creates it, on a host-only stand-in state
        // (no device memory): same schedule, same lowering, same generated tile passes
        sv_state host{};
        host.n = p.n;
        host.g = g;
        host.nloc = p.n - g;
        host.world = world;
        host.rank = 0;
        host.phys.resize(p.n);
        for (int q = 0; q < p.n; q++) host.phys[q] = q;
        CompileOptions hco = hhl_compile_opts(opt, &p, g);
        std::string jitlog;
        hco.dry_run = opt && opt->tile_jit > 0;
        hco.dry_log = &jitlog;
        if (const char *e = getenv("HHLSV_EMU_DIR")) hco.emu_dir = e;     // test tooling (tests/jit_emulator.py)
        Schedule s;
        if (hco.dry_run) {
            std::unique_ptr<sv_program> prog(program_create(&host, fused, factors.empty() ? nullptr : &factors, hco,
                                                            n_logical));
            s = prog->sched;
        } else {
            std::vector<int> phys(p.n);
            for (int q = 0; q < p.n; q++) phys[q] = q;
            if (!hco.phys_init.empty()) phys = hco.phys_init;
            s = compile(fused, factors.empty() ? nullptr : &factors, p.n, p.n - g, phys, hco);
        }
        if (rep) {
            report_plan(rep, p);
            rep->n_logical = n_logical;
            rep->n_fused = s.n_fused;
            rep->n_passes = s.n_passes;
            rep->alg_bytes = s.alg_bytes;
            rep->pass_bytes = s.pass_bytes;
            rep->fusion_kmax_used = fc.kmax;
            rep->model_ms = std::isnan(fc.model_ms) ? schedule_cost_ms(s, p.n - g) : fc.model_ms;
        }
        if (buf && buf_len) {
            std::string t = "INIT_FACTORS " + std::to_string(factors.size()) + "\n" + dump_schedule(s) + jitlog;
            t += "FINAL_MAP";
            for (int q = 0; q < p.n; q++) t += " " + std::to_string(s.phys_out[q]);
            t += "\n";
            size_t n = std::min(buf_len - 1, t.size());
            std::memcpy(buf, t.data(), n);
            buf[n] = 0;
        }
    });
}

sv_status hhl_readout(sv_state *sv, const hhl_report *rep, int N, double *x_out, double *p_success) {
    return guard([&] {
        if (!sv || !rep) fail(SV_E_ARG, "null argument");
        readout(sv, rep, N, x_out, p_success);
    });
}

sv_status hhl_solve(const double *A, const double *b, int N, int clock_qubits, const hhl_options *opt,
                    const sv_dist *dist, void *cuda_stream, double *x_out, hhl_report *rep) {
    return guard([&] {
        if (!x_out) fail(SV_E_ARG, "null x_out");
        hhl_options o{};
        if (opt) o = *opt;
        if (clock_qubits > 0) o.clock_qubits = clock_qubits;
        if (!opt) o.recip_snap = -1.0;
        prof_mark("hhl_solve start");
        const double tf0 = now_s();
        HHLPlanHost p = plan_of(A, b, N, &o);
        const double t_plan = now_s() - tf0;
        prof_mark("hhl_plan");
        // the HHL program starts with its own initialisation step: no |0...0> fill needed
        sv_state *sv = state_create(p.n, dist, (cudaStream_t)cuda_stream, false);
        prof_mark("state_create");
        sv_program *prog = nullptr;
        try {
            hhl_report r{};
            prog = build_hhl(sv, p, &o, &r, now_s() - t_plan, true);      // front end = plan + build
            const double t0 = now_s();
            program_run(sv, prog);
            if (prof_on()) {
                cudaStreamSynchronize(sv->stream);
                prof_mark("  program_run");
            }
            // norm and P(ancilla = 1) (logical qubit n-1): fused into the last tile pass when the program
            // has it (single GPU, JIT), else one marginal reduction over the state
            double pa[2] = {0.0, 0.0};
            const int anc = p.n - 1;
            if (prog->d_mred) {
                cuda_check(cudaMemcpyAsync(pa, prog->d_mred + 2 * sv_program::kMredCtas, sizeof pa,
                                           cudaMemcpyDeviceToHost, sv->stream),
                           "marginal d2h");
                cuda_check(cudaStreamSynchronize(sv->stream), "marginal sync");
            } else {
                state_probabilities(sv, &anc, 1, pa);
            }
            r.norm2 = pa[0] + pa[1];
            r.p_anc1 = pa[1];
            prof_mark("  norm + P(ancilla)");
            readout(sv, &r, N, x_out, &r.p_success);
            r.t_sim_s = now_s() - t0;
            prof_mark("run + readout");
            if (rep) *rep = r;
        } catch (...) {
            program_destroy(prog);
            state_destroy(sv);
            throw;
        }
        program_destroy(prog);
        state_destroy(sv);
        prof_mark("destroy");
    });
}

}  // extern "C"
