/*
 * CPU ORACLE -- test infrastructure only.
 *
 * A plain-C restatement of the reference's compiled CONCORD sweep kernels
 * (/root/reference/pkg/src/parconcord/_ckernels.pyx) used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * Nothing in the product path (paper_2106_09382_b200/) links or calls this.
 *
 * Arithmetic is deliberately identical to the reference build
 * (gcc -O3, x86-64 baseline, no FMA, sequential scalar sums):
 *   - dot products run u = 0..p-1 in order with separate mul and add,
 *   - compiled with -ffp-contract=off so no fused multiply-add appears,
 * which makes every sweep bitwise equal to the reference's `compiled`
 * backend (pinned against tests/golden/ and oracle/_ref in tests).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* _ckernels.pyx:18-22 */
static inline double soft(double x, double tau) {
    double a = fabs(x) - tau;
    if (a <= 0.0) return 0.0;
    return x > 0.0 ? a : -a;
}

/* _ckernels.pyx:25-38: closed-form minimiser for the symmetric pair (r, s). */
static inline double offdiag_value(const double* om, const double* t, int64_t p,
                                   int64_t r, int64_t s, double shrink) {
    const double* omr = om + r * p;
    const double* oms = om + s * p;
    const double* tr = t + r * p;
    const double* ts = t + s * p;
    double s1 = 0.0, s2 = 0.0;
    for (int64_t u = 0; u < p; ++u) s1 += omr[u] * ts[u];
    for (int64_t u = 0; u < p; ++u) s2 += oms[u] * tr[u];
    double num = -(s1 + s2 - omr[s] * (ts[s] + tr[r]));
    return soft(num, shrink) / (tr[r] + ts[s]);
}

/* _ckernels.pyx:41-50: positive root of the diagonal stationarity condition. */
static inline double diag_value(const double* om, const double* t, int64_t p,
                                int64_t i, double n) {
    const double* omi = om + i * p;
    const double* ti = t + i * p;
    double a = 0.0;
    for (int64_t u = 0; u < p; ++u) a += omi[u] * ti[u];
    a -= omi[i] * ti[i];
    return (-a + sqrt(a * a + 4.0 * n * ti[i])) / (2.0 * ti[i]);
}

/* _ckernels.pyx:53-65: serial cycle, upper triangle row-major, then diagonals. */
void oracle_cd_sweep(double* om, const double* t, int64_t p, double n, double shrink) {
    for (int64_t r = 0; r < p; ++r)
        for (int64_t s = r + 1; s < p; ++s) {
            double v = offdiag_value(om, t, p, r, s, shrink);
            om[r * p + s] = v;
            om[s * p + r] = v;
        }
    for (int64_t i = 0; i < p; ++i) om[i * p + i] = diag_value(om, t, p, i, n);
}

/* _ckernels.pyx:68-102: rounds of concurrent pair updates, then diagonals.
 * Pairs in one round share no index, so the parallel loop is bitwise equal
 * to the serial one for every thread count. */
void oracle_pcd_sweep(double* om, const double* t, int64_t p, double n, double shrink,
                      const int64_t* rs, const int64_t* ss, const int64_t* offsets,
                      int64_t nrounds, int workers) {
    if (workers < 1) workers = 1;
    for (int64_t k = 0; k < nrounds; ++k) {
        int64_t lo = offsets[k], hi = offsets[k + 1];
#pragma omp parallel for schedule(static) num_threads(workers) if (workers > 1)
        for (int64_t idx = lo; idx < hi; ++idx) {
            double v = offdiag_value(om, t, p, rs[idx], ss[idx], shrink);
            om[rs[idx] * p + ss[idx]] = v;
            om[ss[idx] * p + rs[idx]] = v;
        }
    }
#pragma omp parallel for schedule(static) num_threads(workers) if (workers > 1)
    for (int64_t i = 0; i < p; ++i) om[i * p + i] = diag_value(om, t, p, i, n);
}

/* _ckernels.pyx:105-118: serial replay of the flattened schedule. */
void oracle_u2_sweep(double* om, const double* t, int64_t p, double n, double shrink,
                     const int64_t* rs, const int64_t* ss, int64_t m) {
    for (int64_t idx = 0; idx < m; ++idx) {
        double v = offdiag_value(om, t, p, rs[idx], ss[idx], shrink);
        om[rs[idx] * p + ss[idx]] = v;
        om[ss[idx] * p + rs[idx]] = v;
    }
    for (int64_t i = 0; i < p; ++i) om[i * p + i] = diag_value(om, t, p, i, n);
}

/* schedule.py:68-88 (build_circle_schedule) + solver.py:166-178
 * (_flatten_schedule): the round-robin rotation, phantom pairs dropped,
 * 0-based (r < s) in the reference's within-round order q = 0..half-1.
 * rs/ss need room for p*(p-1)/2 entries, offsets for p_even entries.
 * Returns the number of rounds (p_even - 1). */
int64_t oracle_circle_flat(int64_t p, int64_t* rs, int64_t* ss, int64_t* offsets) {
    int64_t pe = p + (p % 2), half = pe / 2, cnt = 0;
    int64_t* j = (int64_t*)malloc(sizeof(int64_t) * pe);
    for (int64_t i = 0; i < pe; ++i) j[i] = i + 1;
    offsets[0] = 0;
    for (int64_t k = 0; k < pe - 1; ++k) {
        for (int64_t q = 0; q < half; ++q) {
            int64_t a = j[q], b = j[pe - 1 - q];
            int64_t r = a < b ? a : b, s = a < b ? b : a;
            if (s > p) continue; /* phantom (schedule.py:49-55) */
            rs[cnt] = r - 1;
            ss[cnt] = s - 1;
            ++cnt;
        }
        offsets[k + 1] = cnt;
        int64_t tmp = j[pe - 1];
        memmove(j + 2, j + 1, sizeof(int64_t) * (pe - 2));
        j[1] = tmp;
    }
    free(j);
    return pe - 1;
}

/* model.py:210-217 restated without a p^3 GEMM for large p is NOT done here:
 * the objective stays in numpy (oracle.py) exactly as the reference has it. */

/* max |a-b| over the upper triangle incl. diagonal (solver.py:141-163,187-189;
 * the halving tree equals a linear scan because max/abs do not round). */
double oracle_vech_max_abs_diff(const double* a, const double* b, int64_t p) {
    double worst = 0.0;
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = i; j < p; ++j) {
            double d = fabs(a[i * p + j] - b[i * p + j]);
            if (d > worst) worst = d;
        }
    return worst;
}
