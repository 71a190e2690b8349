// Host front end: gate validation, the HHL circuit builder and the fusion pass.
//
// HHL builder — PAPER.md:156-199 ("Practical HHL procedures" box), Fig. 5 (conceptual
// circuit), resources formula PAPER.md:225-242, with the qlsarepo
// settings the paper defers to as read in DESIGN.md R1-R17. This is the
// paper's own "future work" item: native (C++) QPE/HHL circuit generation,
// replacing Python generation that was "the current bottleneck".
//
// Fusion — PAPER.md:128 §II-C and Fig. 4: merge applicable gates into
// one fused gate. B200 mode: sequential greedy, structure preserving (dense stays dense
// up to kmax targets, diagonal stays diagonal up to diag_kmax qubits, controlled ops with
// equal controls merge their target blocks), SWAPs seen through by relabelling.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>

#include "jit.h"
#include "sv_internal.h"

namespace hhlsv {

// ------------------------------------------------------------------ errors ----
void fail(sv_status code, const std::string &msg) { throw Error{code, msg}; }

bool prof_on() {
    static const bool on = getenv("HHLSV_PROFILE") != nullptr;
    return on;
}

void prof_mark(const char *stage) {
    if (!prof_on()) return;
    using clk = std::chrono::steady_clock;
    static thread_local clk::time_point last = clk::now();
    const auto now = clk::now();
    fprintf(stderr, "[hhlsv] %-28s %8.3f ms\n", stage, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

double alg_bytes(const Gate &g, int n) {
    const double full = 32.0 * std::ldexp(1.0, n);     // read + write 16 B per amplitude
    switch (g.kind) {
        case Kind::Controlled: return full / std::ldexp(1.0, (int)g.controls.size());
        case Kind::Swap: return 0.0;
        default: return full;
    }
}

static void check_qubits(const std::vector<int> &q, int n, const char *what) {
    for (size_t i = 0; i < q.size(); i++) {
        if (q[i] < 0 || q[i] >= n) fail(SV_E_ARG, std::string(what) + ": qubit index out of range");
        for (size_t j = 0; j < i; j++)
            if (q[i] == q[j]) fail(SV_E_ARG, std::string(what) + ": duplicated qubit");
    }
}

static double unitarity_defect(const std::vector<cplx> &U, int d) {
    double worst = 0.0;
    for (int r = 0; r < d; r++)
        for (int c = 0; c < d; c++) {
            cplx acc = 0;
            for (int k = 0; k < d; k++) acc += U[r * d + k] * std::conj(U[c * d + k]);
            if (r == c) acc -= 1.0;
            worst = std::max(worst, std::abs(acc));
        }
    return worst;
}

Gate gate_from_abi(const sv_gate &a, int n) {
    Gate g;
    if (a.kind < SV_DENSE || a.kind > SV_SWAP) fail(SV_E_ARG, "unknown gate kind");
    g.kind = (Kind)a.kind;
    if (a.n_targets < 1 || (a.n_targets > 0 && !a.targets)) fail(SV_E_ARG, "gate needs targets");
    if (a.n_controls < 0 || (a.n_controls > 0 && !a.controls)) fail(SV_E_ARG, "bad controls");
    for (int i = 0; i < a.n_targets; i++) g.targets.push_back(a.targets[i]);
    for (int i = 0; i < a.n_controls; i++) g.controls.push_back(a.controls[i]);
    g.cvals = a.control_values;
    std::vector<int> all = g.targets;
    all.insert(all.end(), g.controls.begin(), g.controls.end());
    check_qubits(all, n, "gate");
    const int k = a.n_targets;
    switch (g.kind) {
        case Kind::Dense:
        case Kind::Controlled: {
            if (k > 5) fail(SV_E_ARG, "dense/controlled gates take at most 5 targets");
            if (g.kind == Kind::Dense && !g.controls.empty()) fail(SV_E_ARG, "dense gate with controls");
            if (g.kind == Kind::Controlled && (g.controls.empty() || g.controls.size() > 20))
                fail(SV_E_ARG, "controlled gate needs 1..20 controls");
            if (!a.data) fail(SV_E_ARG, "gate matrix missing");
            const int d = 1 << k;
            g.data.resize((size_t)d * d);
            for (size_t i = 0; i < g.data.size(); i++) g.data[i] = cplx(a.data[2 * i], a.data[2 * i + 1]);
            if (unitarity_defect(g.data, d) > 1e-10) fail(SV_E_NOTUNITARY, "gate matrix is not unitary (1e-10)");
            break;
        }
        case Kind::Diagonal: {
            if (k > 12) fail(SV_E_ARG, "diagonal gates take at most 12 qubits");
            if (!g.controls.empty()) fail(SV_E_ARG, "diagonal gate with controls");
            if (!a.data) fail(SV_E_ARG, "diagonal table missing");
            g.data.resize((size_t)1 << k);
            for (size_t i = 0; i < g.data.size(); i++) g.data[i] = cplx(a.data[2 * i], a.data[2 * i + 1]);
            for (auto &z : g.data)
                if (std::abs(std::abs(z) - 1.0) > 1e-10) fail(SV_E_NOTUNITARY, "diagonal entry not unimodular");
            break;
        }
        case Kind::RecipRY: {
            if (k != 1) fail(SV_E_ARG, "recip_ry has exactly one target (the ancilla)");
            if (g.controls.empty() || g.controls.size() > 62) fail(SV_E_ARG, "recip_ry needs 1..62 clock qubits");
            if (!(a.recip_delta >= 0.0) || !std::isfinite(a.recip_delta)) fail(SV_E_ARG, "bad recip_delta");
            g.delta = a.recip_delta;
            g.is_signed = a.recip_signed ? 1 : 0;
            g.snap = a.recip_snap > 0 ? a.recip_snap : 0.0;
            break;
        }
        case Kind::Swap:
            if (k != 2 || !g.controls.empty()) fail(SV_E_ARG, "swap takes exactly two targets");
            break;
    }
    return g;
}

// ------------------------------------------------------------ eigensolver ----
// Cyclic Jacobi for a real symmetric N×N matrix (row-major in A). Eigenvalues ascending,
// eigenvectors as columns of V (column-major V[i + N*s]).
void jacobi_eigh(int N, std::vector<double> A, std::vector<double> &lam, std::vector<double> &V) {
    std::vector<double> Q((size_t)N * N, 0.0);
    for (int i = 0; i < N; i++) Q[(size_t)i * N + i] = 1.0;   // row-major Q, columns = eigvecs
    auto a = [&](int i, int j) -> double & { return A[(size_t)i * N + j]; };
    double prev_off = INFINITY;
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < N; i++)
            for (int j = 0; j < N; j++) {
                tot += a(i, j) * a(i, j);
                if (i != j) off += a(i, j) * a(i, j);
            }
        // converged, or the off-diagonal mass stopped shrinking (rounding floor reached): a fixed
        // 1e-34 relative target alone could spin all 100 sweeps at the floor (4 ms at N = 32)
        if (off <= 1e-34 * tot || off == 0.0 || off >= prev_off) break;
        prev_off = off;
        for (int p = 0; p < N - 1; p++)
            for (int q = p + 1; q < N; q++) {
                double apq = a(p, q);
                if (apq == 0.0) continue;
                double app = a(p, p), aqq = a(q, q);
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < N; k++) {           // A <- J^T A J
                    double akp = a(k, p), akq = a(k, q);
                    a(k, p) = c * akp - s * akq;
                    a(k, q) = s * akp + c * akq;
                }
                for (int k = 0; k < N; k++) {
                    double apk = a(p, k), aqk = a(q, k);
                    a(p, k) = c * apk - s * aqk;
                    a(q, k) = s * apk + c * aqk;
                }
                for (int k = 0; k < N; k++) {
                    double qkp = Q[(size_t)k * N + p], qkq = Q[(size_t)k * N + q];
                    Q[(size_t)k * N + p] = c * qkp - s * qkq;
                    Q[(size_t)k * N + q] = s * qkp + c * qkq;
                }
            }
    }
    std::vector<int> order(N);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
    lam.resize(N);
    V.assign((size_t)N * N, 0.0);
    for (int s = 0; s < N; s++) {
        lam[s] = a(order[s], order[s]);
        for (int i = 0; i < N; i++) V[i + (size_t)N * s] = Q[(size_t)i * N + order[s]];
    }
}

// ------------------------------------------------------------------- HHL ----
// Step 1 of the procedure box: normalise b, expand to a power of two
// (identity padding, R9); eigen-analysis; n_QPE from the resources formula read per
// F3 (R2/R3: +1 sign qubit always); delta and t per qlsarepo (R4); phi_s per R13.
HHLPlanHost hhl_plan(const double *A, const double *b, int N0, int clock_qubits, double snap, const double *eig_lam,
                     const double *eig_V) {
    if (!A || !b || N0 < 1) fail(SV_E_ARG, "hhl: null A/b or N < 1");
    HHLPlanHost p;
    p.n_orig = N0;
    bool symmetric = true;
    for (int i = 0; i < N0; i++)
        for (int j = 0; j < N0; j++)
            if (std::fabs(A[i * N0 + j] - A[j * N0 + i]) > 1e-10) symmetric = false;
    double bn = 0.0;
    for (int i = 0; i < N0; i++) bn += b[i] * b[i];
    bn = std::sqrt(bn);
    if (!(bn > 0.0)) fail(SV_E_ARG, "hhl: b is zero");
    int nb = 1;
    while ((1 << nb) < N0) nb++;
    int Np = 1 << nb;
    // step 1(b): identity padding; step 1(c): [[0, A], [A^T, 0]] [0; x] = [b; 0] when A is not
    // symmetric, after the expansion (Table 1's 30-bus* n_data = 6)
    std::vector<double> Ap((size_t)Np * Np, 0.0);
    for (int i = 0; i < Np; i++) Ap[(size_t)i * Np + i] = 1.0;
    for (int i = 0; i < N0; i++)
        for (int j = 0; j < N0; j++) Ap[(size_t)i * Np + j] = A[i * N0 + j];
    int N = Np;
    if (!symmetric) {
        nb += 1;
        N = 2 * Np;
        p.x_offset = Np;
    }
    p.N = N;
    p.n_b = nb;
    p.A.assign((size_t)N * N, 0.0);
    if (symmetric) {
        p.A = Ap;
    } else {
        for (int i = 0; i < Np; i++)
            for (int j = 0; j < Np; j++) {
                p.A[(size_t)i * N + (Np + j)] = Ap[(size_t)i * Np + j];
                p.A[(size_t)(Np + j) * N + i] = Ap[(size_t)i * Np + j];
            }
    }
    p.b_hat.assign(N, 0.0);
    for (int i = 0; i < N0; i++) p.b_hat[i] = b[i] / bn;
    p.b_norm = bn;
    if (!eig_lam != !eig_V) fail(SV_E_ARG, "hhl: eig_lambda and eig_vectors must be given together");
    if (eig_lam) {
        // caller-supplied eigendecomposition (hhl_options.eig_*): row-major V, column s <-> lambda_s
        p.lam.assign(eig_lam, eig_lam + N);
        p.V.assign((size_t)N * N, 0.0);
        double lmax = 1.0;
        for (int s = 0; s < N; s++) lmax = std::max(lmax, std::fabs(p.lam[s]));
        for (int i = 0; i < N; i++)
            for (int s = 0; s < N; s++) p.V[i + (size_t)N * s] = eig_V[(size_t)i * N + s];
        for (int s = 0; s < N; s++) {
            for (int i = 0; i < N; i++) {
                double av = 0.0;
                for (int j = 0; j < N; j++) av += p.A[(size_t)i * N + j] * p.V[j + (size_t)N * s];
                if (!(std::fabs(av - p.lam[s] * p.V[i + (size_t)N * s]) <= 1e-8 * lmax))
                    fail(SV_E_ARG, "hhl: eig_vectors/eig_lambda do not diagonalise the padded A");
            }
            for (int r = 0; r < N; r++) {
                double d = 0.0;
                for (int i = 0; i < N; i++) d += p.V[i + (size_t)N * s] * p.V[i + (size_t)N * r];
                if (!(std::fabs(d - (r == s ? 1.0 : 0.0)) <= 1e-10)) fail(SV_E_ARG, "hhl: eig_vectors not orthonormal");
            }
        }
    } else {
        jacobi_eigh(N, p.A, p.lam, p.V);
    }
    p.lam_min = INFINITY;
    p.lam_max = 0.0;
    for (double l : p.lam) {
        p.lam_min = std::min(p.lam_min, std::fabs(l));
        p.lam_max = std::max(p.lam_max, std::fabs(l));
    }
    if (!(p.lam_min > 0.0)) fail(SV_E_ARG, "hhl: A is singular");
    p.kappa = p.lam_max / p.lam_min;
    int nc = clock_qubits;
    if (nc <= 0) nc = std::max(nb + 1, (int)std::ceil(std::log2(p.kappa + 1.0))) + 1;
    if (nc < 2 || nc > 60) fail(SV_E_ARG, "hhl: clock register size out of range");
    p.n_c = nc;
    p.n = nb + nc + 1;
    const int n_l = nc - 1;
    double lt = std::fabs(p.lam_min * (std::ldexp(1.0, n_l) - 1.0) / p.lam_max);
    if (std::fabs(lt - 1.0) < 1e-7) lt = 1.0;
    p.delta = std::ldexp(std::floor(lt), -n_l);
    if (p.delta == 0.0) fail(SV_E_CLOCK, "hhl: clock register too small for kappa (delta = 0)");
    p.t = 2.0 * M_PI * p.delta / p.lam_min / 2.0;
    p.phi.resize(N);
    for (int s = 0; s < N; s++) p.phi[s] = (p.lam[s] / p.lam_min) * (p.delta / 2.0);
    p.snap = snap;
    return p;
}

static std::vector<cplx> hadamard() {
    const double h = 1.0 / std::sqrt(2.0);
    return {h, h, h, -h};
}

// Textbook QFT on `q` (q[0] = LSB): for j = n-1..0: H(q_j), CP(pi/2^(j-k)) for k = j-1..0;
// then swaps q_i <-> q_{n-1-i}. Inverse: reversed list, conjugated phases (R12).
static void append_qft(std::vector<Gate> &out, const std::vector<int> &q, bool inverse) {
    std::vector<Gate> l;
    const int n = (int)q.size();
    for (int j = n - 1; j >= 0; j--) {
        Gate h;
        h.kind = Kind::Dense;
        h.targets = {q[j]};
        h.data = hadamard();
        l.push_back(h);
        for (int k = j - 1; k >= 0; k--) {
            Gate cp;
            cp.kind = Kind::Diagonal;
            cp.targets = {q[j], q[k]};
            double th = M_PI / std::ldexp(1.0, j - k);
            cp.data = {1.0, 1.0, 1.0, std::polar(1.0, th)};
            l.push_back(cp);
        }
    }
    for (int i = 0; i < n / 2; i++) {
        Gate s;
        s.kind = Kind::Swap;
        s.targets = {q[i], q[n - 1 - i]};
        l.push_back(s);
    }
    if (inverse) {
        std::reverse(l.begin(), l.end());
        for (auto &g : l)
            if (g.kind == Kind::Diagonal)
                for (auto &z : g.data) z = std::conj(z);
    }
    out.insert(out.end(), l.begin(), l.end());
}

// Fig. 5 circuit: U_b; H^{(x)n_c}; c-U_j (j ascending); IQFT; RECIP_RY;
// QFT; c-U_j^dagger (j descending); H^{(x)n_c}. U_j = V diag(exp(2 pi i frac(2^j phi_s))) V^T.
// Eigenbasis form of the controlled-evolution chain:
//   prod_j c-U_j = (V (x) I) D (V^T (x) I),  D[s, m] = exp(2 pi i sum_j m_j frac(2^j phi_s)),
// emitted as V^T on the system register, then one diagonal table per chunk of clock bits
// (system qubits + up to 4 clock qubits). The inverse chain is D^dagger then V.
static void append_eigen_chain(std::vector<Gate> &g, const HHLPlanHost &p, const std::vector<int> &sys,
                               const std::vector<int> &clk, bool inverse) {
    // forward chain: V^T, D ; inverse chain: D^dagger, V. The V closing the forward chain and the
    // V^T opening the inverse chain cancel (V V^T = I): everything between them (IQFT, RECIP_RY,
    // QFT) acts on clock/ancilla qubits only and commutes with V (x) I.
    const int N = p.N, nb = p.n_b, nc = p.n_c;
    auto dense_V = [&](bool transpose) {
        Gate v;
        v.kind = Kind::Dense;
        v.targets = sys;
        v.data.assign((size_t)N * N, 0.0);
        for (int r = 0; r < N; r++)
            for (int c = 0; c < N; c++)
                v.data[(size_t)r * N + c] = transpose ? p.V[c + (size_t)N * r] : p.V[r + (size_t)N * c];
        return v;
    };
    // One factor per clock bit: D_j = diag over (system, clock bit j), 2^(n_b+1) entries. Fusion
    // leaves them separate (HHL fusion caps diagonal merging at a few qubits), so the tile
    // scheduler can place each factor in whichever pass holds its clock bit's QFT Hadamard; the
    // factors of one register phase are then merged after scheduling (compile.cpp
    // merge_phase_diagonals). Lets the final V join the last QFT pass.
    const int chunk = jit_config().eigen_chunk > 0 ? jit_config().eigen_chunk : 1;   // experiments
    std::vector<Gate> diags;
    for (int j0 = 0; j0 < nc; j0 += chunk) {
        const int cj = std::min(chunk, nc - j0);
        Gate d;
        d.kind = Kind::Diagonal;
        d.targets = sys;
        for (int j = 0; j < cj; j++) d.targets.push_back(clk[j0 + j]);
        d.data.resize((size_t)N << cj);
        for (size_t mc = 0; mc < ((size_t)1 << cj); mc++)
            for (int s = 0; s < N; s++) {
                double acc = 0.0;
                for (int j = 0; j < cj; j++)
                    if ((mc >> j) & 1) {
                        double x = std::ldexp(p.phi[s], j0 + j);
                        acc += x - std::floor(x);
                    }
                acc -= std::floor(acc);
                d.data[s + (mc << nb)] = std::polar(1.0, (inverse ? -2.0 : 2.0) * M_PI * acc);
            }
        diags.push_back(std::move(d));
    }
    if (!inverse) g.push_back(dense_V(true));            // V^T
    for (auto &d : diags) g.push_back(std::move(d));
    if (inverse) g.push_back(dense_V(false));            // V
}

std::vector<Gate> hhl_build(const HHLPlanHost &p, int qpe_mode) {
    const int N = p.N, nb = p.n_b, nc = p.n_c;
    std::vector<int> sys(nb), clk(nc);
    std::iota(sys.begin(), sys.end(), 0);
    std::iota(clk.begin(), clk.end(), nb);
    const int anc = nb + nc;
    std::vector<Gate> g;
    {   // Householder state preparation U_b = I - 2 v v^T/(v^T v), v = e0 - b_hat (R11)
        Gate u;
        u.kind = Kind::Dense;
        u.targets = sys;
        u.data.assign((size_t)N * N, 0.0);
        std::vector<double> v(p.b_hat);
        for (auto &x : v) x = -x;
        v[0] += 1.0;
        double vv = 0.0;
        for (double x : v) vv += x * x;
        for (int r = 0; r < N; r++)
            for (int c = 0; c < N; c++)
                u.data[(size_t)r * N + c] = (r == c ? 1.0 : 0.0) - (vv > 1e-300 ? 2.0 * v[r] * v[c] / vv : 0.0);
        g.push_back(u);
    }
    for (int j = 0; j < nc; j++) {
        Gate h;
        h.kind = Kind::Dense;
        h.targets = {clk[j]};
        h.data = hadamard();
        g.push_back(h);
    }
    if (qpe_mode == 1) {
        append_eigen_chain(g, p, sys, clk, false);
        append_qft(g, clk, true);
        Gate r;
        r.kind = Kind::RecipRY;
        r.targets = {anc};
        r.controls = clk;
        r.delta = p.delta;
        r.is_signed = 1;
        r.snap = p.snap;
        g.push_back(r);
        append_qft(g, clk, false);
        append_eigen_chain(g, p, sys, clk, true);
        for (int j = 0; j < nc; j++) {
            Gate h;
            h.kind = Kind::Dense;
            h.targets = {clk[j]};
            h.data = hadamard();
            g.push_back(h);
        }
        return g;
    }
    std::vector<std::vector<cplx>> U(nc);
    for (int j = 0; j < nc; j++) {
        std::vector<cplx> ph(N);
        for (int s = 0; s < N; s++) {
            double x = std::ldexp(p.phi[s], j);
            double f = x - std::floor(x);
            ph[s] = std::polar(1.0, 2.0 * M_PI * f);
        }
        U[j].assign((size_t)N * N, 0.0);
        for (int r = 0; r < N; r++)
            for (int c = 0; c < N; c++) {
                cplx acc = 0;
                for (int s = 0; s < N; s++) acc += p.V[r + (size_t)N * s] * ph[s] * p.V[c + (size_t)N * s];
                U[j][(size_t)r * N + c] = acc;
            }
    }
    for (int j = 0; j < nc; j++) {
        Gate c;
        c.kind = Kind::Controlled;
        c.targets = sys;
        c.controls = {clk[j]};
        c.cvals = 1;
        c.data = U[j];
        g.push_back(c);
    }
    append_qft(g, clk, true);
    {
        Gate r;
        r.kind = Kind::RecipRY;
        r.targets = {anc};
        r.controls = clk;
        r.delta = p.delta;
        r.is_signed = 1;
        r.snap = p.snap;
        g.push_back(r);
    }
    append_qft(g, clk, false);
    for (int j = nc - 1; j >= 0; j--) {
        Gate c;
        c.kind = Kind::Controlled;
        c.targets = sys;
        c.controls = {clk[j]};
        c.cvals = 1;
        c.data.assign((size_t)N * N, 0.0);
        for (int r = 0; r < N; r++)
            for (int cc = 0; cc < N; cc++) c.data[(size_t)r * N + cc] = std::conj(U[j][(size_t)cc * N + r]);
        g.push_back(c);
    }
    for (int j = 0; j < nc; j++) {
        Gate h;
        h.kind = Kind::Dense;
        h.targets = {clk[j]};
        h.data = hadamard();
        g.push_back(h);
    }
    return g;
}

static std::vector<cplx> embed_dense(const std::vector<cplx> &m, const std::vector<int> &q,
                                     const std::vector<int> &u);

// ------------------------------------------------------------ product fold ----
size_t fold_product_prefix(const std::vector<Gate> &gates, int n, std::vector<ProductFactor> &factors,
                           bool fold_diagonals) {
    std::vector<char> touched(n, 0);
    const bool diag_phase = false;
    factors.clear();
    size_t i = 0;
    for (; i < gates.size(); i++) {
        const Gate &g = gates[i];
        if (g.kind != Kind::Dense) break;
        if (diag_phase) break;
        bool fresh = true;
        for (int q : g.targets) fresh &= !touched[q];
        if (!fresh) {
            // a dense gate acting inside ONE existing factor: multiply it into that factor
            ProductFactor *host = nullptr;
            for (auto &f : factors) {
                bool inside = true;
                for (int q : g.targets) inside &= std::find(f.qubits.begin(), f.qubits.end(), q) != f.qubits.end();
                if (inside) host = &f;
            }
            if (!host) break;
            const size_t d = host->vec.size();
            auto E = embed_dense(g.data, g.targets, host->qubits);
            std::vector<cplx> nv(d, 0.0);
            for (size_t r = 0; r < d; r++)
                for (size_t c = 0; c < d; c++) nv[r] += E[r * d + c] * host->vec[c];
            host->vec.swap(nv);
            continue;
        }
        ProductFactor f;
        f.qubits = g.targets;
        const size_t d = (size_t)1 << g.targets.size();
        f.vec.resize(d);
        for (size_t r = 0; r < d; r++) f.vec[r] = g.data[r * d];     // column 0: U|0>
        for (int q : g.targets) touched[q] = 1;
        factors.push_back(std::move(f));
    }
    // diagonal gates right after the product state: folded as per-amplitude phase tables
    for (; fold_diagonals && i < gates.size(); i++) {
        const Gate &g = gates[i];
        if (g.kind != Kind::Diagonal || g.targets.size() > 12) break;
        size_t nd = 0;
        for (auto &f : factors) nd += f.diag;
        if (nd >= 8) break;
        ProductFactor f;
        f.qubits = g.targets;
        f.vec = g.data;
        f.diag = true;
        factors.push_back(std::move(f));
    }
    return i;
}

// ------------------------------------------------------------------ fusion ----
// Embed matrix m acting on qubit list q (q[0] = LSB) into the 2^|u| space of list u.
static std::vector<cplx> embed_dense(const std::vector<cplx> &m, const std::vector<int> &q,
                                     const std::vector<int> &u) {
    const size_t du = (size_t)1 << u.size();
    std::vector<int> pos(q.size());
    uint64_t qmask = 0;
    for (size_t i = 0; i < q.size(); i++) {
        pos[i] = (int)(std::find(u.begin(), u.end(), q[i]) - u.begin());
        qmask |= 1ull << pos[i];
    }
    const size_t dq = (size_t)1 << q.size();
    auto sub = [&](size_t x) {
        size_t s = 0;
        for (size_t i = 0; i < q.size(); i++)
            if ((x >> pos[i]) & 1) s |= (size_t)1 << i;
        return s;
    };
    std::vector<cplx> E(du * du, 0.0);
    for (size_t r = 0; r < du; r++)
        for (size_t c = 0; c < du; c++)
            if ((r & ~qmask) == (c & ~qmask)) E[r * du + c] = m[sub(r) * dq + sub(c)];
    return E;
}


static std::vector<cplx> matmul(const std::vector<cplx> &a, const std::vector<cplx> &b, size_t d) {
    std::vector<cplx> c(d * d, 0.0);
    for (size_t i = 0; i < d; i++)
        for (size_t k = 0; k < d; k++) {
            const cplx aik = a[i * d + k];
            if (aik == 0.0) continue;
            for (size_t j = 0; j < d; j++) c[i * d + j] += aik * b[k * d + j];
        }
    return c;
}

static std::vector<int> union_of(const std::vector<int> &a, const std::vector<int> &b) {
    std::vector<int> u = a;
    for (int x : b)
        if (std::find(u.begin(), u.end(), x) == u.end()) u.push_back(x);
    return u;
}

static bool disjoint(const std::vector<int> &a, const std::vector<int> &b) {
    for (int x : a)
        if (std::find(b.begin(), b.end(), x) != b.end()) return false;
    return true;
}

// Try to merge `nx` (applied after `cur`) into `cur`. Returns true on success.
bool merge_diagonal(Gate &cur, const Gate &nx, int diag_kmax) {
    auto u = union_of(cur.targets, nx.targets);
    if ((int)u.size() > diag_kmax) return false;
    // cur.targets is a prefix of u: its table tiles over the appended bits; nx's bits are
    // gathered per entry (few bits for the CP ladders being merged)
    const size_t du = (size_t)1 << u.size(), mc = cur.data.size() - 1;
    std::vector<int> pos(nx.targets.size());
    for (size_t i = 0; i < nx.targets.size(); i++)
        pos[i] = (int)(std::find(u.begin(), u.end(), nx.targets[i]) - u.begin());
    std::vector<cplx> a(du);
    for (size_t x = 0; x < du; x++) {
        size_t j = 0;
        for (size_t i = 0; i < pos.size(); i++)
            if ((x >> pos[i]) & 1) j |= (size_t)1 << i;
        a[x] = cur.data[x & mc] * nx.data[j];
    }
    cur.targets = u;
    cur.data = std::move(a);
    return true;
}

static bool try_merge(Gate &cur, const Gate &nx, const FuseOptions &o) {
    if (cur.kind == Kind::RecipRY || nx.kind == Kind::RecipRY) return false;
    if (cur.kind == Kind::Diagonal && nx.kind == Kind::Diagonal) return merge_diagonal(cur, nx, o.diag_kmax);
    const bool cd = cur.kind == Kind::Dense || cur.kind == Kind::Diagonal;
    const bool nd = nx.kind == Kind::Dense || nx.kind == Kind::Diagonal;
    if (cd && nd) {
        auto u = union_of(cur.targets, nx.targets);
        if ((int)u.size() > o.kmax) return false;
        auto to_dense = [](const Gate &g) {
            if (g.kind == Kind::Dense) return g.data;
            const size_t d = g.data.size();
            std::vector<cplx> m(d * d, 0.0);
            for (size_t i = 0; i < d; i++) m[i * d + i] = g.data[i];
            return m;
        };
        auto a = embed_dense(to_dense(cur), cur.targets, u);
        auto b = embed_dense(to_dense(nx), nx.targets, u);
        cur.data = matmul(b, a, (size_t)1 << u.size());
        cur.targets = u;
        cur.kind = Kind::Dense;
        return true;
    }
    if (cur.kind == Kind::Controlled && nx.kind == Kind::Controlled && cur.controls == nx.controls &&
        cur.cvals == nx.cvals) {
        auto u = union_of(cur.targets, nx.targets);
        if ((int)u.size() > o.kmax || !disjoint(u, cur.controls)) return false;
        auto a = embed_dense(cur.data, cur.targets, u), b = embed_dense(nx.data, nx.targets, u);
        cur.data = matmul(b, a, (size_t)1 << u.size());
        cur.targets = u;
        return true;
    }
    return false;
}

// ---------------------------------------------------- paper mode (Fig. 4) ----
// SV-Sim's gate fusion as PAPER.md:207 (Fig. 4 caption) describes it, for "applicable gates" (one-
// and two-qubit gates): four strategies applied with priority (1) consecutive one-qubit gates on the
// same qubit are fused; then (2) a one-qubit gate is absorbed into the two-qubit gate that follows it
// on its qubit, and (3) into the one that precedes it; finally (4) consecutive two-qubit gates on the
// same qubit pair are fused. "Consecutive" = no other gate touches those qubits in between (gates on
// other qubits commute with them). Wider gates and the reciprocal rotation are kept as they are and
// block fusion across them. Diagonal stays diagonal when both parts are diagonal.
static bool applicable(const Gate &g) {
    if (g.kind == Kind::Dense || g.kind == Kind::Diagonal) return g.targets.size() <= 2;
    if (g.kind == Kind::Controlled) return g.targets.size() == 1 && g.controls.size() == 1;
    return false;
}
static std::vector<int> qubits_of(const Gate &g) { return union_of(g.targets, g.controls); }
static Gate as_plain(const Gate &g) {      // controlled 1+1 -> dense 4x4 on {target, control}
    if (g.kind != Kind::Controlled) return g;
    Gate d;
    d.kind = Kind::Dense;
    d.targets = {g.targets[0], g.controls[0]};
    d.data.assign(16, 0.0);
    const int want = (int)(g.cvals & 1);
    for (int c = 0; c < 2; c++)
        for (int r = 0; r < 2; r++)
            for (int k = 0; k < 2; k++)
                d.data[(size_t)((c << 1) | r) * 4 + ((c << 1) | k)] = (c == want) ? g.data[r * 2 + k] : cplx(r == k ? 1.0 : 0.0);
    return d;
}
// b applied after a (both applicable, plain): the fused gate on the union of their qubits
static Gate compose(const Gate &a, const Gate &b) {
    Gate r;
    if (a.kind == Kind::Diagonal && b.kind == Kind::Diagonal) {
        r = a;
        merge_diagonal(r, b, 64);
        return r;
    }
    auto dense = [](const Gate &g) {
        if (g.kind == Kind::Dense) return g.data;
        const size_t d = g.data.size();
        std::vector<cplx> m(d * d, 0.0);
        for (size_t i = 0; i < d; i++) m[i * d + i] = g.data[i];
        return m;
    };
    r.kind = Kind::Dense;
    r.targets = union_of(a.targets, b.targets);
    const auto ea = embed_dense(dense(a), a.targets, r.targets), eb = embed_dense(dense(b), b.targets, r.targets);
    r.data = matmul(eb, ea, (size_t)1 << r.targets.size());
    return r;
}
static std::vector<Gate> fuse_paper(std::vector<Gate> g) {
    for (auto &x : g)
        if (applicable(x)) x = as_plain(x);
    std::vector<char> dead(g.size(), 0);
    auto touches = [&](size_t i, int q) {
        auto v = qubits_of(g[i]);
        return std::find(v.begin(), v.end(), q) != v.end();
    };
    auto next_on = [&](size_t i, int q) -> long {      // next live gate touching q after i
        for (size_t j = i + 1; j < g.size(); j++)
            if (!dead[j] && touches(j, q)) return (long)j;
        return -1;
    };
    auto prev_on = [&](size_t i, int q) -> long {
        for (long j = (long)i - 1; j >= 0; j--)
            if (!dead[j] && touches((size_t)j, q)) return j;
        return -1;
    };
    auto is1 = [&](size_t i) { return !dead[i] && applicable(g[i]) && qubits_of(g[i]).size() == 1; };
    auto is2 = [&](size_t i) { return !dead[i] && applicable(g[i]) && qubits_of(g[i]).size() == 2; };
    // (1) one-qubit + one-qubit
    for (size_t i = 0; i < g.size(); i++) {
        if (!is1(i)) continue;
        const long j = next_on(i, g[i].targets[0]);
        if (j >= 0 && is1((size_t)j)) {
            g[j] = compose(g[i], g[j]);
            dead[i] = 1;
        }
    }
    // (2) one-qubit into the following two-qubit gate, (3) into the preceding one
    for (size_t i = 0; i < g.size(); i++) {
        if (!is1(i)) continue;
        const long j = next_on(i, g[i].targets[0]);
        if (j >= 0 && is2((size_t)j)) {
            g[j] = compose(g[i], g[j]);
            dead[i] = 1;
        }
    }
    for (size_t i = 0; i < g.size(); i++) {
        if (!is1(i)) continue;
        const long j = prev_on(i, g[i].targets[0]);
        if (j >= 0 && is2((size_t)j)) {
            g[j] = compose(g[j], g[i]);
            dead[i] = 1;
        }
    }
    // (4) two-qubit + two-qubit on the same pair
    for (size_t i = 0; i < g.size(); i++) {
        if (!is2(i)) continue;
        auto qi = qubits_of(g[i]);
        const long j0 = next_on(i, qi[0]), j1 = next_on(i, qi[1]);
        if (j0 >= 0 && j0 == j1 && is2((size_t)j0)) {
            auto qj = qubits_of(g[j0]);
            if ((qj[0] == qi[0] && qj[1] == qi[1]) || (qj[0] == qi[1] && qj[1] == qi[0])) {
                g[j0] = compose(g[i], g[j0]);
                dead[i] = 1;
            }
        }
    }
    std::vector<Gate> out;
    for (size_t i = 0; i < g.size(); i++)
        if (!dead[i]) out.push_back(std::move(g[i]));
    return out;
}

std::vector<Gate> fuse(const std::vector<Gate> &in, const FuseOptions &o) {
    // Relabel through SWAPs: name[q] = the qubit that currently holds original wire q's role.
    int nq = 0;
    for (auto &g : in) {
        for (int q : g.targets) nq = std::max(nq, q + 1);
        for (int q : g.controls) nq = std::max(nq, q + 1);
    }
    std::vector<int> where(nq);
    std::iota(where.begin(), where.end(), 0);   // logical wire -> position after pending swaps
    std::vector<Gate> out;
    Gate cur;
    bool have = false;
    auto flush = [&]() {
        if (have) out.push_back(std::move(cur));
        have = false;
    };
    for (const Gate &g0 : in) {
        if (g0.kind == Kind::Swap) {
            std::swap(where[g0.targets[0]], where[g0.targets[1]]);
            continue;
        }
        Gate g = g0;
        for (int &q : g.targets) q = where[q];
        for (int &q : g.controls) q = where[q];
        if (o.kmax <= 0 || o.mode == 1) {
            out.push_back(std::move(g));
            continue;
        }
        if (have && try_merge(cur, g, o)) continue;
        flush();
        cur = std::move(g);
        have = true;
    }
    flush();
    if (o.mode == 1) out = fuse_paper(std::move(out));
    // Realise the accumulated relabelling as trailing swaps (executed as relabels, free).
    std::vector<int> pos = where;               // wire w sits at position pos[w]
    for (int w = 0; w < nq; w++) {
        if (pos[w] == w) continue;
        int v = (int)(std::find(pos.begin(), pos.end(), w) - pos.begin());   // wire v sits at position w
        Gate s;
        s.kind = Kind::Swap;
        s.targets = {w, pos[w]};
        out.push_back(s);
        // swapping positions w and pos[w]: wire v moves to pos[w], wire w moves to w
        pos[v] = pos[w];
        pos[w] = w;
    }
    return out;
}

}  // namespace hhlsv
