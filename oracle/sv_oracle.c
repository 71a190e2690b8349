/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU state-vector simulator for the HHL hot path
 * of arXiv 2402.08136 ("the unitary evolution of the state", §II-C;
 * "the statevector of |psi> can be read directly", §III-A step 3).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library. It shares no code, header, table or
 * helper with the CUDA product in paper_2402_08136_b200/.
 *
 * Conventions (R1): amplitudes are complex128
 * stored interleaved (re, im); qubit q is bit q of the amplitude index
 * (little-endian); for a k-qubit gate, targets[0] is the least-significant bit of
 * the matrix row/column index; matrices are row-major.
 *
 * Each gate is applied exactly as its plain definition states: a loop over all
 * 2^n indices, acting once per group (the index whose target bits are all 0),
 * gathering the 2^k amplitudes of the group, multiplying by the gate matrix and
 * scattering back. fp64, no blocking, no fusion.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;

#define ORC_MAXK 10

/* Controlled dense gate: psi <- (|c><c| ⊗ U + (I - |c><c|) ⊗ I) psi, with
 * control qubits `controls[j]` required to equal bit j of `cvals`.
 * n_controls = 0 is an unconditioned dense gate. Returns 0, or -1 on bad args. */
int orc_apply_controlled(int n, double *psi_il, int k, const int *targets, int n_controls,
                         const int *controls, uint64_t cvals, const double *U_il) {
    if (k < 1 || k > ORC_MAXK || n < k + n_controls) return -1;
    cplx *psi = (cplx *)psi_il;
    const cplx *U = (const cplx *)U_il;
    const uint64_t dim = 1ull << k;
    uint64_t tmask = 0, cmask = 0, cwant = 0;
    for (int i = 0; i < k; i++) tmask |= 1ull << targets[i];
    for (int j = 0; j < n_controls; j++) {
        cmask |= 1ull << controls[j];
        if ((cvals >> j) & 1ull) cwant |= 1ull << controls[j];
    }
    const uint64_t N = 1ull << n;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)N; ii++) {
        uint64_t base = (uint64_t)ii;
        if (base & tmask) continue;              /* not a group representative */
        if ((base & cmask) != cwant) continue;   /* control not satisfied: identity */
        cplx vin[1 << ORC_MAXK];
        uint64_t idx[1 << ORC_MAXK];
        for (uint64_t r = 0; r < dim; r++) {
            uint64_t a = base;
            for (int i = 0; i < k; i++)
                if ((r >> i) & 1ull) a |= 1ull << targets[i];
            idx[r] = a;
            vin[r] = psi[a];
        }
        for (uint64_t r = 0; r < dim; r++) {
            cplx acc = 0;
            for (uint64_t c = 0; c < dim; c++) acc += U[r * dim + c] * vin[c];
            psi[idx[r]] = acc;
        }
    }
    return 0;
}

/* Diagonal gate: psi_i <- d[bits(i, qubits)] psi_i (bit j of the table index = qubits[j]).
 * Plain definition of a diagonal unitary (the CP ladders of the (I)QFT are diagonal). */
int orc_apply_diagonal(int n, double *psi_il, int k, const int *qubits, const double *d_il) {
    if (k < 1 || k > 30 || n < k) return -1;
    cplx *psi = (cplx *)psi_il;
    const cplx *d = (const cplx *)d_il;
    const uint64_t N = 1ull << n;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)N; ii++) {
        uint64_t v = 0;
        for (int j = 0; j < k; j++)
            if (((uint64_t)ii >> qubits[j]) & 1ull) v |= 1ull << j;
        psi[ii] *= d[v];
    }
    return 0;
}

/* Eigenvalue-inversion rotation (the uniformly-controlled RY of Fig. 5,
 * PAPER.md:212-217, built "following the settings in [qlsarepo]").
 * For clock value m = sum_j bit(clock[j]) 2^j (LSB first) and half-range
 * L = 2^(n_c - signed):
 *   m' = m            if !signed or m <  2^(n_c-1)
 *   m' = 2^n_c - m    (negative eigenvalue, sign -1) otherwise
 *   r  = delta * L / m'   (m' = 0 -> s = 0)
 *   s  = 1 if |r - 1| <= snap ; r if r < 1 ; 0 otherwise;   s <- sign * s
 *   theta = 2 asin(s);  RY(theta) = [[cos th/2, -sin th/2], [sin th/2, cos th/2]]
 * applied to the ancilla pair (anc = 0, anc = 1). SURVEY §8(c) "reference
 * conventions", R4/R6. */
double orc_recip_s(uint64_t m, int n_c, double delta, int is_signed, double snap) {
    if (m == 0) return 0.0;
    double sign = 1.0;
    uint64_t mp = m;
    if (is_signed && m >= (1ull << (n_c - 1))) {
        mp = (1ull << n_c) - m;
        sign = -1.0;
    }
    double L = ldexp(1.0, n_c - (is_signed ? 1 : 0));
    double r = delta * L / (double)mp;
    double s;
    if (fabs(r - 1.0) <= snap) s = 1.0;
    else if (r < 1.0) s = r;
    else s = 0.0;
    return sign * s;
}

int orc_apply_recip_ry(int n, double *psi_il, int anc, int n_c, const int *clock, double delta,
                       int is_signed, double snap) {
    if (n_c < 1 || n_c > 62 || anc < 0 || anc >= n) return -1;
    cplx *psi = (cplx *)psi_il;
    const uint64_t N = 1ull << n;
    const uint64_t abit = 1ull << anc;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)N; ii++) {
        uint64_t i0 = (uint64_t)ii;
        if (i0 & abit) continue;
        uint64_t m = 0;
        for (int j = 0; j < n_c; j++)
            if ((i0 >> clock[j]) & 1ull) m |= 1ull << j;
        double s = orc_recip_s(m, n_c, delta, is_signed, snap);
        double theta = 2.0 * asin(s);
        double c2 = cos(theta / 2.0), s2 = sin(theta / 2.0);
        cplx x0 = psi[i0], x1 = psi[i0 | abit];
        psi[i0] = c2 * x0 - s2 * x1;
        psi[i0 | abit] = s2 * x0 + c2 * x1;
    }
    return 0;
}

/* Marginal probabilities over `qubits` (bit j of the output index = qubits[j]):
 * out[v] = sum over i with bits(i, qubits) = v of |psi_i|^2. Sequential sum in
 * index order ("P(measure ancilla and get 1)"). */
int orc_marginal(int n, const double *psi_il, int nq, const int *qubits, double *out) {
    if (nq < 0 || nq > 30) return -1;
    const cplx *psi = (const cplx *)psi_il;
    memset(out, 0, sizeof(double) << nq);
    const uint64_t N = 1ull << n;
    for (uint64_t i = 0; i < N; i++) {
        uint64_t v = 0;
        for (int j = 0; j < nq; j++)
            if ((i >> qubits[j]) & 1ull) v |= 1ull << j;
        double a = creal(psi[i]), b = cimag(psi[i]);
        out[v] += a * a + b * b;
    }
    return 0;
}

/* |0...0> initialisation. */
void orc_init_zero(int n, double *psi_il) {
    memset(psi_il, 0, sizeof(double) * 2 * (1ull << n));
    psi_il[0] = 1.0;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
