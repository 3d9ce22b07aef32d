// Shared device helpers for the CONCORD-PCD sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace concord {

// ---------------------------------------------------------------------------
// Circle-method 1-factorisation (schedule.py:68-88) in closed form.
// 0-based ids, p_even = p + p%2, m = p_even - 1 rounds, round k in [0, m).
// Position 0 holds id 0; position i>=1 holds 1 + ((i - 1 - k) mod m); round k
// pairs position q with position m - q.  Solving for the partner gives
//   x >= 1:  y = 1 + ((-x - 1 - 2k) mod m),  partner = (y == x) ? 0 : y
//   x == 0:  partner = 1 + ((m - 1 - k) mod m)
// (verified against the reference rotation in tests/test_schedule.py).
// Odd p: id p is the phantom; pairs touching it are skipped (schedule.py:49-55).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int circle_partner(int x, int k, int m) {
    // division-free for 0 <= k < m, 0 <= x <= m: m-1-k is in [0, m) and 3m-x-1-2k in [1, 3m-2]
    if (x == 0) return m - k;
    int t = 3 * m - x - 1 - 2 * k;
    t -= (t >= 2 * m) ? 2 * m : ((t >= m) ? m : 0);
    const int y = 1 + t;
    return (y == x) ? 0 : y;
}

// Pair q (0 <= q < p_even/2) of round k, returned with r < s.
__host__ __device__ __forceinline__ void circle_pair(int k, int q, int m, int& r, int& s) {
    int a, b;
    if (q == 0) {
        a = 0;
        b = 1 + (m - 1 - k) % m;
    } else {
        a = 1 + (q - 1 - k + m) % m;
        b = 1 + (2 * m - q - 1 - k) % m;
    }
    r = a < b ? a : b;
    s = a < b ? b : a;
}

// Soft threshold exactly as _ckernels.pyx:18-22 (exact 0.0 inside the band).
__device__ __forceinline__ double soft_threshold(double x, double tau) {
    double a = __dsub_rn(fabs(x), tau);
    if (a <= 0.0) return 0.0;
    return x > 0.0 ? a : -a;
}

// Off-diagonal closed form (_ckernels.pyx:37-38) from the two half sums
// s1 = sum_u om[r,u] t[s,u], s2 = sum_u om[s,u] t[r,u].  No FMA contraction.
__device__ __forceinline__ double offdiag_from_sums(double s1, double s2, double om_rs,
                                                    double t_rr, double t_ss, double shrink) {
    double num = -__dsub_rn(__dadd_rn(s1, s2), __dmul_rn(om_rs, __dadd_rn(t_ss, t_rr)));
    return __ddiv_rn(soft_threshold(num, shrink), __dadd_rn(t_rr, t_ss));
}

// Diagonal closed form (_ckernels.pyx:49-50) from dot = sum_u om[i,u] t[i,u].
__device__ __forceinline__ double diag_from_dot(double dot, double om_ii, double t_ii, double n) {
    double a = __dsub_rn(dot, __dmul_rn(om_ii, t_ii));
    double disc = __dadd_rn(__dmul_rn(a, a), __dmul_rn(__dmul_rn(4.0, n), t_ii));
    return __ddiv_rn(__dadd_rn(-a, __dsqrt_rn(disc)), __dmul_rn(2.0, t_ii));
}

// Pair q of round k without integer division: c1 = m - 1 - k (common.cuh has the closed form).
__device__ __forceinline__ void round_pair(int q, int m, int c1, int& r, int& s) {
    int a, b;
    if (q == 0) {
        a = 0;
        b = 1 + c1;
    } else {
        const int t = q + c1;
        const int u = m + c1 - q;
        a = 1 + (t >= m ? t - m : t);
        b = 1 + (u >= m ? u - m : u);
    }
    r = min(a, b);
    s = max(a, b);
}

// delta of pair (r, s) from the published half values vr = (W[s,r], Om[s,r]),
// vs = (W[r,s], Om[r,s]); same operation order as offdiag_from_sums, with the
// division skipped when the soft threshold returns its exact 0.0.
__device__ __forceinline__ double pair_delta(double2 vr, double2 vs, double trr, double tss, double shrink,
                                             double& nv) {
    const double om = vs.y;
    const double num = -__dsub_rn(__dadd_rn(vs.x, vr.x), __dmul_rn(om, __dadd_rn(tss, trr)));
    const double av = __dsub_rn(fabs(num), shrink);
    nv = (av <= 0.0) ? 0.0 : __ddiv_rn(num > 0.0 ? av : -av, __dadd_rn(trr, tss));
    return __dsub_rn(nv, om);
}

// Row published for column c in phase ph (ph < m: colour ph, ph == m: diagonal), or -1.
__device__ __forceinline__ int pub_row(int ph, int c, int m, int p) {
    const int x = (ph < m) ? circle_partner(c, ph, m) : c;
    return x < p ? x : -1;
}

// Row whose value moves row x in phase ph (its pair partner; x itself on the diagonal).
__device__ __forceinline__ int src_row(int ph, int x, int m) { return ph < m ? circle_partner(x, ph, m) : x; }

// ---------------------------------------------------------------------------
// Grid-wide barrier for a cooperative (co-resident) launch: one monotonic
// 64-bit arrival counter, zeroed by the host before each launch.  `target` is
// (barrier ordinal) * gridDim.x.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1ull);
        while (ld_acquire_u64(ctr) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Watchdog of every spin loop of the fit kernels: a wait that lasts kHangNs turns into a
// diagnostic line and a trap (a launch error on the host) instead of a hung device.
constexpr unsigned long long kHangNs = 20ull * 1000ull * 1000ull * 1000ull;

// The report goes to mapped host memory (readable after the trap): what, CTA, block, values.
__device__ __forceinline__ void hang_report(long long* hang, int what, int blk, long long v0, long long v1,
                                            long long v2, long long v3) {
    volatile long long* h = hang;
    h[1] = blockIdx.x;
    h[2] = blk;
    h[3] = v0;
    h[4] = v1;
    h[5] = v2;
    h[6] = v3;
    __threadfence_system();
    h[0] = what + 1;
    __threadfence_system();
    __trap();
}


// |delta| for the convergence max, with NaN mapped to +inf: fmax / warp_max drop a NaN
// operand, and the reference's np.max(np.abs(...)) (solver.py:141-163) never converges on one.
__device__ __forceinline__ double abs_delta(double d) {
    return (d != d) ? __longlong_as_double(0x7ff0000000000000ll) : fabs(d);
}

__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace concord
