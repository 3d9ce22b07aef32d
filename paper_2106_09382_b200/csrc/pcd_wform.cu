// Persistent cooperative CONCORD-PCD fit kernel (W-form), sm_100a.
//
// Replaces the reference's per-iteration loop pcd_fit (solver.py:254-294) over
// the compiled sweep pcd_sweep (_ckernels.pyx:68-102).  Instead of the two
// length-p dot products per pair (_ckernels.pyx:33-36, 16p^3 bytes per
// sweep) it maintains W = Omega * T on the device:
//   s1 = sum_u om[r,u] t[s,u] = W[r,s],   s2 = sum_u om[s,u] t[r,u] = W[s,r]
// and after a pair changes by d applies the two row streams
//   W[r,:] += d * T[s,:],   W[s,:] += d * T[r,:]
// (diagonal i: W[i,:] += d_i * T[i,:]).  Exact zeros from the soft threshold
// make most d exactly 0, and those rows are skipped exactly.
//
// Layout in HBM: T, W and dense Omega are column-block ("slab") major.  CTA b
// owns columns [b*w, b*w+w); slab b is a p x w row-major block, so every row
// stream only touches the CTA's own slab.
//
// Phases.  A sweep is m = p_even-1 colour phases then the diagonal phase
// (_ckernels.pyx:81-102); phases are numbered globally, g = sweep*(m+1) + ph.
// Each CTA runs two warp-specialised roles:
//
//  * chain warps (WFORM_CHAIN_WARPS): the latency-critical colour chain.  Per
//    phase g: wait on the grid barrier (all publishes of g visible); publish
//    (W[x,c], Om[x,c]) of every own column c for phase g+1 (x = partner of c);
//    evaluate this CTA's 1/nblk share of the colour-g closed forms
//    (_ckernels.pyx:25-38) and write the per-row deltas (dring) and the
//    non-zero (r, s, delta, new) list; arrive.  One grid barrier per phase.
//  * apply warps (the rest): stream the delta lists into the own slab -- in
//    phase order, batched over up to WFORM_BATCH phases, trailing the chain by
//    up to `lmax` phases -- and the dense diagonal step (also folding in the
//    objective trace, model.py:210-217).  After each batch they stage, in
//    shared memory, the W/Om cells the next publishes need together with the
//    T entries of the phases they have not applied yet.
//
// A publish therefore starts from a staged value W[x,c] that includes every
// phase <= C (the apply watermark) and brings it forward with
//   W[x,c] = fma(d_k, T[src_k(x), c], W[x,c])   for k = C+1 .. g, d_k != 0
// -- the very operations, in the very order, the apply warps perform on the
// slab -- so every published value is bitwise the value of the sequential
// W-form.  d_k comes from dring for k < g and is recomputed from the phase-g
// publish buffer for k = g.  Every CTA sees identical values, so the max
// |delta| convergence metric (solver.py:287) needs no extra reduction.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "pcd_wform.h"

namespace concord {

// Loops over the shard copies of the exchange buffers with compile-time indices
// (the pointer arrays stay in the kernel-parameter bank instead of a local copy).
#define FOR_COPIES(r) _Pragma("unroll") for (int r = 0; r < WFORM_MAX_SHARDS; ++r) if (r < G)
#define FOR_COPIES_A(r) _Pragma("unroll") for (int r = 0; r < WFORM_MAX_SHARDS; ++r) if (r < a.G)

constexpr int kThreads = WFORM_THREADS;
constexpr int kChainWarps = WFORM_CHAIN_WARPS;
constexpr int kChain = kChainWarps * 32;
constexpr int kApply = kThreads - kChain;
constexpr int kApplyWarps = kApply / 32;
constexpr int kPairCap = WFORM_PAIR_CAP;
constexpr int kBatch = WFORM_BATCH;
constexpr int kSlots = WFORM_STAGE_SLOTS;
constexpr int kMaxLag = WFORM_MAX_LAG;
constexpr int kUnroll = 2;
#ifndef WFORM_ROW_UNROLL
#define WFORM_ROW_UNROLL 2
#endif
constexpr int kRowUnroll = WFORM_ROW_UNROLL;  // row-stream items in flight per thread (bytes in flight / SM)

// Phase-ph delta of row x (paired with y) recomputed from that phase's publish buffer.
__device__ __forceinline__ double row_delta(int ph, int x, int y, const double2* pb, const double* tdiag, int m,
                                            double shrink, double n) {
    double nv;
    if (ph < m) {
        const int r = min(x, y), s = max(x, y);
        return pair_delta(ldcg2(pb + r), ldcg2(pb + s), __ldg(tdiag + r), __ldg(tdiag + s), shrink, nv);
    }
    const double2 v = ldcg2(pb + x);
    nv = diag_from_dot(v.x, v.y, __ldg(tdiag + x), n);
    return __dsub_rn(nv, v.y);
}

__device__ __forceinline__ void bar_chain() { asm volatile("bar.sync 1, %0;" ::"n"(kChain) : "memory"); }
__device__ __forceinline__ void bar_apply() { asm volatile("bar.sync 2, %0;" ::"n"(kApply) : "memory"); }

__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_vol(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

// Exclusive scan of s[0..n) in place by the apply warps; returns the total (also in s[n]).
__device__ int apply_scan(int* s, int n, int ta, int* s_wsum) {
    const int lane = ta & 31, wa = ta >> 5;
    const int per = (n + kApply - 1) / kApply;
    const int lo = min(n, ta * per), hi = min(n, lo + per);
    int local = 0;
    for (int i = lo; i < hi; ++i) local += s[i];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[wa] = incl;
    bar_apply();
    int wbase = 0, total = 0;
    for (int j = 0; j < kApplyWarps; ++j) {
        const int v = s_wsum[j];
        if (j < wa) wbase += v;
        total += v;
    }
    int run = wbase + incl - local;
    for (int i = lo; i < hi; ++i) {
        const int v = s[i];
        s[i] = run;
        run += v;
    }
    if (ta == 0) s[n] = total;
    bar_apply();
    return total;
}

// Row streams of delta-list entries [e_lo, e_hi) (shared-memory indices; only
// batch phase `only` when only >= 0): W[dst, own] = fma(d, T[src, own], W[dst, own])
// for both rows of every pair.
__device__ __forceinline__ void apply_rows(const int2* L_rs, const double* L_d, const int* L_ph, int only, int e_lo,
                                           int e_hi, int w2, double* __restrict__ Wb, const double* __restrict__ Tb,
                                           int ta) {
    const int w = 2 * w2;
    const int per = 2 * w2;
    const int items = (e_hi - e_lo) * per;
    // item idx = ta + (k * kRowUnroll + u) * kApply -> (entry q, position rem), stepped without division
    const int dq = kApply / per, dr = kApply - dq * per;
    int q = ta / per, rem = ta - (ta / per) * per;
    for (int base = 0; base < items; base += kApply * kRowUnroll) {
        double2 tv[kRowUnroll], wv[kRowUnroll];
        double2* wp[kRowUnroll];
        double dd[kRowUnroll];
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) {
            const int idx = base + u * kApply + ta;
            wp[u] = nullptr;
            if (idx < items) {
                const int e = e_lo + q;
                if (only < 0 || L_ph[e] == only) {
                    const int h = rem >= w2;
                    const int j2 = rem - h * w2;
                    const int2 rs = L_rs[e];
                    dd[u] = L_d[e];
                    const int dst = h ? rs.y : rs.x;
                    const int src = h ? rs.x : rs.y;
                    wp[u] = reinterpret_cast<double2*>(Wb + (long long)dst * w) + j2;
                    tv[u] = __ldcg(reinterpret_cast<const double2*>(Tb + (long long)src * w) + j2);
                    wv[u] = __ldcg(wp[u]);
                }
            }
            q += dq;
            rem += dr;
            if (rem >= per) {
                rem -= per;
                ++q;
            }
        }
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) {
            if (wp[u]) {
                wv[u].x = fma(dd[u], tv[u].x, wv[u].x);
                wv[u].y = fma(dd[u], tv[u].y, wv[u].y);
                *wp[u] = wv[u];
            }
        }
    }
}

// Arrive on the grid barrier of every shard: make this CTA's exchange-buffer
// stores visible (GPU scope, or system scope when the shards are separate
// GPUs reached over NVLink), then bump every copy of the arrival counter.
__device__ __forceinline__ void arrive_all(const WformArgs& a) {
    if (a.sys_scope) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        FOR_COPIES_A(r) asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(a.x.bar[r]) : "memory");
    } else if (a.G == 1) {
        // release-reduction: MEMBAR.ALL.GPU + REDG (no sequentially-consistent fence, no L1 invalidate)
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.x.bar[0]) : "memory");
    } else {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        FOR_COPIES_A(r) asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(a.x.bar[r]) : "memory");
    }
}

// Wait until the barrier counter reaches `target`: relaxed polling (a plain L2
// load per iteration, no L1 invalidate per poll), then one acquire fence.
__device__ __forceinline__ void wait_counter(const unsigned long long* ctr, unsigned long long target, int sys,
                                             int g, long long* hang) {
    unsigned long long v;
    const unsigned long long t0 = globaltimer_ns();
    int spins = 0;
    do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (++spins == 4096) {
            spins = 0;
            if (globaltimer_ns() - t0 > kHangNs) hang_report(hang, 0, g, (long long)v, (long long)target, 0, 0);
        }
    } while (v < target);
    if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

struct Smem {
    double* stage;  // [kSlots][2 + lmax][w]: W, Om, T of the uncovered phases
    int* s_off;     // [kBatch * nblk + 1]
    int2* L_rs;     // [kPairCap]
    double* L_d;    // [kPairCap]  (diag chunk: delta)
    double* L_new;  // [kPairCap]  (diag chunk: new value)
    int* L_ph;      // [kPairCap]  batch phase of each entry
    unsigned* bm;   // [(p + 31) / 32] row bitmap of a chunk (conflict detection)
    double* td;     // [p] T diagonal in shared memory (small p), or NULL
};

// kProf: the phase profiler (CONCORD_PHASE_PROFILE); the production instance carries no timers.
template <bool kProf>
#define PCLK() (kProf ? clock64() : 0ll)
__global__ void __launch_bounds__(kThreads, 1) pcd_wform_kernel(WformArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_epoch;               // chain: last phase g whose barrier was passed
    __shared__ int s_staged;              // apply: highest publish phase staged
    __shared__ int s_stop;                // chain: phase of the final diagonal step, or -1
    __shared__ int s_stbase[kSlots];      // apply watermark each stage slot was taken at
    __shared__ int s_cnt;                 // chain: list compaction counter
    __shared__ int s_conflict;            // apply: a row appears twice in the current chunk
    __shared__ int s_wsum[kApplyWarps];
    __shared__ double s_red[4][kApplyWarps];
    __shared__ int s_iters, s_conv;
    __shared__ int s_aE, s_aStop;         // apply: control state broadcast by apply thread 0
    __shared__ int s_nent, s_multi;       // apply: single-entry segments gathered / a segment had more

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bl = blockIdx.x;        // slab of this launch
    const int b = a.blk0 + bl;        // global CTA = global column block
    const int nblk = a.nblk_tot;
    const int G = a.G;
    const int shard = b / a.nblk_loc;  // whose copy of the exchange buffers is "ours"
    const int p = a.p, m = a.m, w = a.w, w2 = a.w >> 1, half = a.half, lmax = a.lmax;
    const int c0 = b * w;
    const int wl = max(0, min(w, p - c0));
    const int q_lo = min(b * a.share, half), q_hi = min(q_lo + a.share, half);
    double* __restrict__ Wb = a.W + (long long)bl * a.slab;
    const double* __restrict__ Tb = a.T + (long long)bl * a.slab;
    double* __restrict__ Ob = a.Om + (long long)bl * a.slab;
    const double2* pubL = a.x.pub[0];
    const double* dringL = a.x.dring[0];
    const int2* lrsL = a.x.list_rs[0];
    const double2* ldnL = a.x.list_dn[0];
    const int* lcntL = a.x.list_cnt[0];
    unsigned long long* barL = a.x.bar[0];
    const unsigned long long* dmaxL = a.x.dmax[0];
#pragma unroll
    for (int r = 1; r < WFORM_MAX_SHARDS; ++r)
        if (r == shard) {
            pubL = a.x.pub[r];
            dringL = a.x.dring[r];
            lrsL = a.x.list_rs[r];
            ldnL = a.x.list_dn[r];
            lcntL = a.x.list_cnt[r];
            barL = a.x.bar[r];
            dmaxL = a.x.dmax[r];
        }
    const int ssz = (2 + lmax) * w;  // doubles per stage slot
#define TD(i) (sm.td ? sm.td[i] : __ldg(a.tdiag + (i)))

    Smem sm;
    {
        unsigned char* ptr = smem_raw;
        sm.stage = reinterpret_cast<double*>(ptr);
        ptr += sizeof(double) * (size_t)kSlots * ssz;
        sm.L_rs = reinterpret_cast<int2*>(ptr);
        ptr += sizeof(int2) * kPairCap;
        sm.L_d = reinterpret_cast<double*>(ptr);
        ptr += sizeof(double) * kPairCap;
        sm.L_new = reinterpret_cast<double*>(ptr);
        ptr += sizeof(double) * kPairCap;
        sm.L_ph = reinterpret_cast<int*>(ptr);
        ptr += sizeof(int) * kPairCap;
        sm.s_off = reinterpret_cast<int*>(ptr);
        ptr += sizeof(int) * ((size_t)kBatch * nblk + 1);
        sm.bm = reinterpret_cast<unsigned*>(ptr);
        ptr += sizeof(unsigned) * (size_t)((p + 31) / 32);
        ptr = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(ptr) + 15) & ~(uintptr_t)15);
        sm.td = a.tdiag_smem ? reinterpret_cast<double*>(ptr) : nullptr;
    }
    if (sm.td)
        for (int i = tid; i < p; i += kThreads) sm.td[i] = __ldg(a.tdiag + i);
    for (int i = tid; i < (p + 31) / 32; i += kThreads) sm.bm[i] = 0u;

    // ---- initial stages: publish phases 0..min(2, lmax) from the initial W (watermark -1)
    const int init_hi = min(2, lmax);
    for (int idx = tid; idx < (init_hi + 1) * wl; idx += kThreads) {
        const int Q = idx / wl, j = idx - Q * wl;
        const int phQ = Q;  // Q <= 2 <= m except when m == 1 (then lmax == 1 and Q <= 1 <= m)
        const int x = pub_row(phQ, c0 + j, m, p);
        double* st = sm.stage + (size_t)(Q % kSlots) * ssz;
        if (x >= 0) {
            st[j] = Wb[(long long)x * w + j];
            st[w + j] = Ob[(long long)x * w + j];
            for (int i = 0; i < Q; ++i) {  // phases k = 0 .. Q-1 not covered by the stage
                const int y = src_row(i, x, m);
                st[(2 + i) * w + j] = (y < p) ? __ldcg(Tb + (long long)y * w + j) : 0.0;
            }
        }
    }
    if (tid == 0) {
        s_epoch = -1;
        s_staged = init_hi;
        s_stop = -1;
        for (int i = 0; i <= init_hi; ++i) s_stbase[i] = -1;
        s_conflict = 0;
        s_cnt = 0;
    }
    __syncthreads();

    unsigned long long* prof = (kProf && a.prof && bl == 0) ? a.prof : nullptr;

    if (warp < kChainWarps) {
        // ============================================================ chain warps
        const int tc = tid;
        // initial publish (phase 0, no corrections)
        for (int j = tc; j < wl; j += kChain)
            if (pub_row(0, c0 + j, m, p) >= 0) {
                const double2 v = make_double2(sm.stage[j], sm.stage[w + j]);
                FOR_COPIES(r) a.x.pub[r][c0 + j] = v;
            }
        bar_chain();
        if (tc == 0) arrive_all(a);
        if (bl == 0 && tc == 0) a.rec_time[0] = globaltimer_ns();

        int g = 0, ph = 0, it = 0, converged = 0;
        double smax = 0.0;  // max |delta| over this thread's share of the sweep
        int snnz = 0;
        long long t_wait = 0, t_stage = 0, t_work = 0, t_pub = 0, t_share = 0, t_end = 0;
        while (true) {
            long long t0 = PCLK();
            if (tc == 0) {
                const unsigned long long target = a.bar_base + (unsigned long long)(g + 1) * (unsigned long long)nblk;
                wait_counter(barL, target, a.sys_scope, g, a.hang);
                st_vol(&s_epoch, g);
            }
            bar_chain();
            long long t1 = PCLK();
            t_wait += t1 - t0;
            const double2* __restrict__ pb = pubL + (size_t)(g % 3) * p;
            const size_t pn_off = (size_t)((g + 1) % 3) * p;
            const size_t dg_off = (size_t)(g % a.rd) * p;

            bool stop = false;
            if (ph == m) {
                // ---- diagonal step: every CTA evaluates all p closed forms (_ckernels.pyx:41-50)
                double2* dd = a.diagd + (size_t)bl * p;
                double dm = 0.0;
                for (int i = tc; i < p; i += kChain) {
                    const double2 v = ldcg2(pb + i);
                    const double nv = diag_from_dot(v.x, v.y, TD(i), a.n);
                    const double d = __dsub_rn(nv, v.y);
                    dd[i] = make_double2(d, nv);
                    if ((unsigned)(i - c0) < (unsigned)wl)
                        FOR_COPIES(r) a.x.dring[r][dg_off + i] = d;
                    dm = fmax(dm, abs_delta(d));
                }
                dm = warp_max(dm);
                if (lane == 0) s_red[0][warp] = dm;
                bar_chain();
                double dmax_all =
                    __longlong_as_double((long long)__ldcg(dmaxL + (a.it_base + it) % WFORM_DMAX_RING));
                for (int j = 0; j < kChainWarps; ++j) dmax_all = fmax(dmax_all, s_red[0][j]);
                stop = (dmax_all < a.delta_tol) || (it + 1 >= a.max_iter);
                if (bl == 0 && tc == 0) {
                    a.rec_delta[it] = dmax_all;
                    a.rec_time[it + 1] = globaltimer_ns();
                }
                if (b == 0 && tc == 0)  // recycle the accumulator of sweep it+2 (last read at sweep it-2)
                    FOR_COPIES(r) a.x.dmax[r][(a.it_base + it + 2) % WFORM_DMAX_RING] = 0ull;
                if (stop) {
                    converged = dmax_all < a.delta_tol;
                    bar_chain();
                    if (tc == 0) {
                        __threadfence_block();
                        s_iters = it + 1;
                        s_conv = converged;
                        st_vol(&s_stop, g);
                    }
                    break;
                }
            }

            // ---- publish phase g+1: staged value brought forward over the phases it misses
            {
                const int Q = g + 1;
                const int phQ = (ph == m) ? 0 : ph + 1;
                const int slot = Q % kSlots;
                if (tc < wl) {
                    const unsigned long long g0t = globaltimer_ns();
                    while (ld_acquire_cta(&s_staged) < Q) {
                        __nanosleep(20);
                        if (globaltimer_ns() - g0t > kHangNs) hang_report(a.hang, 1, g, Q, ld_vol(&s_staged), 0, 0);
                    }
                }
                long long t2 = PCLK();
                t_stage += t2 - t1;
                t1 = t2;
                const double* st = sm.stage + (size_t)slot * ssz;
                for (int j = tc; j < wl; j += kChain) {
                    const int c = c0 + j;
                    const int x = pub_row(phQ, c, m, p);
                    if (x < 0) continue;
                    // phase-g delta of row x from the phase-g publish buffer (loads issued first)
                    const int y = src_row(ph, x, m);
                    double2 vr = make_double2(0.0, 0.0), vs = vr;
                    if (y < p) {
                        vr = ldcg2(pb + (ph < m ? min(x, y) : x));
                        if (ph < m) vs = ldcg2(pb + max(x, y));
                    }
                    const int C = ld_vol(&s_stbase[slot]);
                    const int L = g - C;  // phases C+1 .. g, L >= 1
                    double dk[kMaxLag];
                    int kslot = (C + 1) % a.rd;
#pragma unroll
                    for (int i = 0; i < kMaxLag; ++i) {
                        dk[i] = (i < L - 1) ? __ldcg(dringL + (size_t)kslot * p + x) : 0.0;
                        kslot = (kslot + 1 == a.rd) ? 0 : kslot + 1;
                    }
                    double dlast = 0.0;
                    if (y < p) {
                        if (ph < m) {
                            const int r = min(x, y), s2 = max(x, y);
                            double nv_;
                            dlast = pair_delta(vr, vs, TD(r), TD(s2), a.shrink, nv_);
                        } else {
                            dlast = __dsub_rn(diag_from_dot(vr.x, vr.y, TD(x), a.n), vr.y);
                        }
                    }
                    double val = st[j];
                    const double om = st[w + j];
#pragma unroll
                    for (int i = 0; i < kMaxLag; ++i)
                        if (i < L - 1 && dk[i] != 0.0) val = fma(dk[i], st[(2 + i) * w + j], val);
                    if (dlast != 0.0) val = fma(dlast, st[(2 + L - 1) * w + j], val);
                    const double2 v = make_double2(val, om);
                    FOR_COPIES(r) a.x.pub[r][pn_off + c] = v;
                }
            }

            if (tc == 0) t_pub += PCLK() - t1;
            // ---- this CTA's share of the colour's closed forms -> dring + delta list segment
            // (runs on the last chain threads, concurrently with the publishers above)
            const int lslot = g % a.rl;
            if (ph < m && b < a.nsh) {
                const int c1 = m - 1 - ph;
                const size_t seg_off = ((size_t)lslot * nblk + b) * a.share;
                const int sid = kChain - 1 - tc;  // share work starts on the last chain warps
                for (int base = q_lo; base < q_hi; base += kChain) {
                    const int q = base + sid;
                    int r = 0, s = 0;
                    double d = 0.0, nv = 0.0;
                    if (q < q_hi) {
                        round_pair(q, m, c1, r, s);
                        if (s < p) {
                            d = pair_delta(ldcg2(pb + r), ldcg2(pb + s), TD(r), TD(s),
                                           a.shrink, nv);
                            FOR_COPIES(c) {
                                a.x.dring[c][dg_off + r] = d;
                                a.x.dring[c][dg_off + s] = d;
                            }
                            if (d != 0.0) {
                                smax = fmax(smax, abs_delta(d));
                                ++snnz;
                            }
                        } else {
                            FOR_COPIES(c) a.x.dring[c][dg_off + r] = 0.0;  // phantom partner (odd p)
                        }
                    }
                    const unsigned mask = __ballot_sync(0xffffffffu, d != 0.0);
                    if (mask) {
                        int basepos = 0;
                        if (lane == 0) basepos = atomicAdd(&s_cnt, __popc(mask));
                        basepos = __shfl_sync(0xffffffffu, basepos, 0);
                        if (d != 0.0) {
                            const int at = basepos + __popc(mask & ((1u << lane) - 1u));
                            FOR_COPIES(c) {
                                a.x.list_rs[c][seg_off + at] = make_int2(r, s);
                                a.x.list_dn[c][seg_off + at] = make_double2(d, nv);
                            }
                        }
                    }
                }
                if (ph == m - 1) {  // this sweep's share statistics: per-warp partials
                    const double mw = warp_max(smax);
                    const double nw = warp_sum((double)snnz);
                    if (lane == 0) {
                        s_red[0][warp] = mw;
                        s_red[1][warp] = nw;
                    }
                    smax = 0.0;
                    snnz = 0;
                }
            }
            if (tc == kChain - 1) t_share += PCLK() - t1;
            const long long tb = PCLK();
            bar_chain();
            if (tc == 0) {
                if (ph < m && b < a.nsh) {
                    FOR_COPIES(r) a.x.list_cnt[r][(size_t)lslot * nblk + b] = s_cnt;
                    s_cnt = 0;
                }
                if (ph == m - 1 && b < a.nsh) {
                    double mb = 0.0, nbk = 0.0;
                    for (int j = 0; j < kChainWarps; ++j) {
                        mb = fmax(mb, s_red[0][j]);
                        nbk += s_red[1][j];
                    }
                    FOR_COPIES(r)
                        atomicMax(a.x.dmax[r] + (a.it_base + it) % WFORM_DMAX_RING,
                                  (unsigned long long)__double_as_longlong(mb));
                    atomicAdd(reinterpret_cast<unsigned long long*>(a.rec_nnz + it), (unsigned long long)nbk);
                }
                arrive_all(a);
            }
            if (tc == 0) t_end += PCLK() - tb;
            t_work += PCLK() - t1;
            if (ph == m) {
                ph = 0;
                ++it;
            } else {
                ++ph;
            }
            ++g;
        }
        if (prof && tc == 0) {
            prof[0] = (unsigned long long)t_wait;
            prof[1] = (unsigned long long)t_stage;
            prof[2] = (unsigned long long)t_work;
            prof[3] = (unsigned long long)g;
            prof[7] = (unsigned long long)t_pub;
            prof[8] = (unsigned long long)t_end;
        }
        if (prof && tc == kChain - 1) {
            prof[9] = (unsigned long long)t_share;
        }
    } else {
        // ============================================================ apply warps
        const int ta = tid - kChain;
        int C = -1;            // every phase <= C is in the own slab
        int cph = m;           // phase-in-sweep of C (C = -1 behaves like a diagonal step)
        int cit = -1;          // sweep of C
        int staged = init_hi;  // highest publish phase staged
        long long t_busy = 0, t_idle = 0, nbatch = 0, t_head = 0, t_diag = 0, t_h0 = 0, t_h1 = 0, t_h2 = 0;
        unsigned long long idle_since = 0;  // watchdog (thread ta == 0)
        while (true) {
            const long long t0 = PCLK();
            bar_apply();  // everyone has consumed the previous broadcast
            if (ta == 0) {
                s_aE = ld_vol(&s_epoch);
                s_aStop = ld_vol(&s_stop);
                s_nent = 0;
                s_multi = 0;
                s_conflict = 0;
                __threadfence_block();
            }
            bar_apply();
            const int E = s_aE;
            const int stopg = s_aStop;
            const int avail = (stopg >= 0) ? stopg : E - 1;  // phases whose deltas are all visible
            const int k0 = C + 1;
            const int ph0 = (cph == m) ? 0 : cph + 1;
            const int it0 = (cph == m) ? cit + 1 : cit;
            const bool have = C < avail;
            const bool diag = have && ph0 == m;
            const int k1 = (have && !diag) ? min(min(avail, k0 + kBatch - 1), k0 + (m - 1 - ph0)) : C;
            const int nb = k1 - C;  // colour phases in this batch (0 for none / diagonal)
            const int nsh = a.nsh;
            const int nseg = nb * nsh;
            // stage with the pre-batch watermark C: the publish corrections cover this batch too
            const int target = (stopg < 0) ? min(E + a.stage_ahead, C + 1 + lmax) : staged;
            const int nq = max(0, target - staged);
            if (!have && nq == 0) {
                t_idle += PCLK() - t0;
                // the chain stopped after this slab already reached the last phase: done
                if (stopg >= 0 && C >= stopg) break;
                if (ta == 0) {
                    if (idle_since == 0) idle_since = globaltimer_ns();
                    else if (globaltimer_ns() - idle_since > kHangNs) hang_report(a.hang, 2, E, C, E, staged, stopg);
                }
                __nanosleep(32);
                continue;
            }
            idle_since = 0;

            const long long ta0 = PCLK();
            // ---- one round trip: segment heads (count + first entry) and the stage cells
            for (int idx = ta; idx < nseg; idx += kApply) {
                const int jb = idx / nsh;
                const int seg = ((k0 + jb) % a.rl) * nblk + (idx - jb * nsh);
                const int cnt = __ldcg(lcntL + seg);
                const int2 rs = __ldcg(lrsL + (size_t)seg * a.share);
                const double2 dn = __ldcg(ldnL + (size_t)seg * a.share);
                sm.s_off[idx] = cnt;
                if (cnt > 1) s_multi = 1;
                if (cnt == 1) {
                    const int pos = atomicAdd(&s_nent, 1);
                    if (pos < kPairCap) {
                        sm.L_rs[pos] = rs;
                        sm.L_d[pos] = dn.x;
                        sm.L_ph[pos] = jb;
                    } else {
                        s_multi = 1;
                    }
                    if ((unsigned)(rs.y - c0) < (unsigned)wl) Ob[(long long)rs.x * w + (rs.y - c0)] = dn.y;
                    if ((unsigned)(rs.x - c0) < (unsigned)wl) Ob[(long long)rs.y * w + (rs.x - c0)] = dn.y;
                }
            }
            const long long ta1 = PCLK();
            for (int idx = ta; idx < nq * wl; idx += kApply) {
                const int qi = idx / wl, j = idx - qi * wl;
                const int Q = staged + 1 + qi;
                const int x = pub_row(Q % (m + 1), c0 + j, m, p);
                if (x < 0) continue;
                double* st = sm.stage + (size_t)(Q % kSlots) * ssz;
                const int L = Q - 1 - C;
                // source rows of phases C+1 .. Q-1 for row x, stepped without integer division
                // (partner_{k+1}(x) = partner_k(x) - 2 mod m for x >= 1, -1 for x == 0)
                int ys[kMaxLag];
                {
                    int phk = ph0;  // phase-in-sweep of C+1
                    int y = (phk < m) ? circle_partner(x, phk, m) : x;
                    const int step = (x == 0) ? 1 : 2;
#pragma unroll
                    for (int i = 0; i < kMaxLag; ++i) {
                        ys[i] = (i < L && y < p) ? y : -1;
                        // advance to phase phk + 1
                        if (phk == m) {
                            phk = 0;
                            y = circle_partner(x, 0, m);
                        } else if (phk == m - 1) {
                            phk = m;
                            y = x;
                        } else {
                            ++phk;
                            if (x == 0) {
                                y = (y == 1) ? m : y - 1;
                            } else {
                                // the self-mapped position becomes 0; undo before stepping
                                int yy = (y == 0) ? x : y;
                                yy -= step;
                                if (yy < 1) yy += m;
                                y = (yy == x) ? 0 : yy;
                            }
                        }
                    }
                }
                double tv[kMaxLag];
#pragma unroll
                for (int i = 0; i < kMaxLag; ++i) tv[i] = __ldcg(Tb + (long long)(ys[i] >= 0 ? ys[i] : x) * w + j);
                const double wv = __ldcg(Wb + (long long)x * w + j);
                const double ov = __ldcg(Ob + (long long)x * w + j);
                st[j] = wv;
                st[w + j] = ov;
#pragma unroll
                for (int i = 0; i < kMaxLag; ++i)
                    if (i < L) st[(2 + i) * w + j] = (ys[i] >= 0) ? tv[i] : 0.0;
            }
            for (int Q = staged + 1 + ta; Q <= target; Q += kApply) s_stbase[Q % kSlots] = C;
            const long long ta2 = PCLK();
            bar_apply();
            t_head += PCLK() - t0;
            t_h0 += ta0 - t0;
            t_h1 += ta1 - ta0;
            t_h2 += ta2 - ta1;
            if (nq > 0) {
                staged = target;
                if (ta == 0) {
                    __threadfence_block();
                    st_vol(&s_staged, staged);
                }
            }

            if (diag) {
                // ---- dense diagonal step over the own slab (+ objective records)
                const double2* dd = a.diagd + (size_t)bl * p;
                double q_acc = 0.0, pen_acc = 0.0, log_acc = 0.0;
                for (int i0 = 0; i0 < p; i0 += kPairCap) {
                    const int iend = min(i0 + kPairCap, p);
                    for (int i = i0 + ta; i < iend; i += kApply) {
                        const double2 v = ldcg2(dd + i);
                        sm.L_d[i - i0] = v.x;
                        sm.L_new[i - i0] = v.y;
                    }
                    bar_apply();
                    const int items = (iend - i0) * w2;
                    for (int base = 0; base < items; base += kApply * kUnroll) {
                        double2 wv[kUnroll], tv[kUnroll], ov[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int idx = base + u * kApply + ta;
                            if (idx < items) {
                                const int ii = idx / w2;
                                const int j2 = idx - ii * w2;
                                const long long off = (long long)(i0 + ii) * w + 2 * j2;
                                wv[u] = __ldcg(reinterpret_cast<const double2*>(Wb + off));
                                if (sm.L_d[ii] != 0.0) tv[u] = __ldcg(reinterpret_cast<const double2*>(Tb + off));
                                if (a.want_trace) ov[u] = *reinterpret_cast<const double2*>(Ob + off);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int idx = base + u * kApply + ta;
                            if (idx < items) {
                                const int ii = idx / w2;
                                const int j2 = idx - ii * w2;
                                const int i = i0 + ii;
                                const long long off = (long long)i * w + 2 * j2;
                                const double d = sm.L_d[ii];
                                if (d != 0.0) {
                                    wv[u].x = fma(d, tv[u].x, wv[u].x);
                                    wv[u].y = fma(d, tv[u].y, wv[u].y);
                                    *reinterpret_cast<double2*>(Wb + off) = wv[u];
                                }
                                const int cj = c0 + 2 * j2;
                                const bool dg0 = (cj == i), dg1 = (cj + 1 == i);
                                if (a.want_trace) {
                                    if (dg0 | dg1) {
                                        if (dg0) ov[u].x = sm.L_new[ii];
                                        if (dg1) ov[u].y = sm.L_new[ii];
                                        *reinterpret_cast<double2*>(Ob + off) = ov[u];
                                        log_acc += log(sm.L_new[ii]);
                                    }
                                    q_acc = fma(wv[u].x, ov[u].x, q_acc);
                                    q_acc = fma(wv[u].y, ov[u].y, q_acc);
                                    if (i < cj) pen_acc += fabs(ov[u].x);
                                    if (i < cj + 1) pen_acc += fabs(ov[u].y);
                                } else if (dg0 | dg1) {
                                    Ob[off + (dg0 ? 0 : 1)] = sm.L_new[ii];
                                }
                            }
                        }
                    }
                    bar_apply();
                }
                if (a.want_trace) {
                    q_acc = warp_sum(q_acc);
                    pen_acc = warp_sum(pen_acc);
                    log_acc = warp_sum(log_acc);
                    const int wa = ta >> 5;
                    if (lane == 0) {
                        s_red[1][wa] = q_acc;
                        s_red[2][wa] = pen_acc;
                        s_red[3][wa] = log_acc;
                    }
                    bar_apply();
                    if (ta == 0) {
                        double v1 = 0.0, v2 = 0.0, v3 = 0.0;
                        for (int j = 0; j < kApplyWarps; ++j) {
                            v1 += s_red[1][j];
                            v2 += s_red[2][j];
                            v3 += s_red[3][j];
                        }
                        double* ro = a.rec_obj + ((size_t)it0 * gridDim.x + bl) * 3;
                        ro[0] = v1;
                        ro[1] = v2;
                        ro[2] = v3;
                    }
                }
                C = k0;
                cph = m;
                cit = it0;
                t_diag += PCLK() - t0;
            } else if (nb > 0) {
                // ---- colour phases k0 .. k1
                int total = 0;
                if (!s_multi) {
                    // every segment had at most one entry: they are already in shared memory
                    const int nent = s_nent;
                    if (nb > 1) {
                        for (int e = ta; e < nent; e += kApply) {
                            const int2 rs = sm.L_rs[e];
                            const unsigned br = 1u << (rs.x & 31), bs = 1u << (rs.y & 31);
                            const unsigned o1 = atomicOr(sm.bm + (rs.x >> 5), br);
                            const unsigned o2 = atomicOr(sm.bm + (rs.y >> 5), bs);
                            if ((o1 & br) | (o2 & bs)) s_conflict = 1;
                        }
                        bar_apply();
                    }
                    if (!s_conflict) {
                        apply_rows(sm.L_rs, sm.L_d, sm.L_ph, -1, 0, nent, w2, Wb, Tb, ta);
                    } else {
                        for (int jb = 0; jb < nb; ++jb) {  // rows repeat across phases: phase by phase
                            apply_rows(sm.L_rs, sm.L_d, sm.L_ph, jb, 0, nent, w2, Wb, Tb, ta);
                            bar_apply();
                        }
                    }
                    bar_apply();
                    if (nb > 1) {
                        for (int e = ta; e < nent; e += kApply) {
                            const int2 rs = sm.L_rs[e];
                            atomicAnd(sm.bm + (rs.x >> 5), ~(1u << (rs.x & 31)));
                            atomicAnd(sm.bm + (rs.y >> 5), ~(1u << (rs.y & 31)));
                        }
                    }
                    total = nent;
                } else {
                    // general path: exclusive scan of the segment counts, entries in phase order
                    total = apply_scan(sm.s_off, nseg, ta, s_wsum);
                    for (int e0 = 0; e0 < total; e0 += kPairCap) {
                        const int e1 = min(total, e0 + kPairCap);
                        for (int e = e0 + ta; e < e1; e += kApply) {
                            int lo = 0, hi = nseg;  // segment: s_off[lo] <= e < s_off[lo+1]
                            while (hi - lo > 1) {
                                const int mid = (lo + hi) >> 1;
                                if (sm.s_off[mid] <= e) lo = mid;
                                else hi = mid;
                            }
                            const int jb = lo / nsh;
                            const int rank = e - sm.s_off[lo];
                            const size_t at =
                                ((size_t)((k0 + jb) % a.rl) * nblk + (lo - jb * nsh)) * a.share + rank;
                            const int2 rs = __ldcg(lrsL + at);
                            const double2 dn = __ldcg(ldnL + at);
                            // segments with one entry had their Omega cells written above
                            if (sm.s_off[lo + 1] - sm.s_off[lo] > 1) {
                                if ((unsigned)(rs.y - c0) < (unsigned)wl) Ob[(long long)rs.x * w + (rs.y - c0)] = dn.y;
                                if ((unsigned)(rs.x - c0) < (unsigned)wl) Ob[(long long)rs.y * w + (rs.x - c0)] = dn.y;
                            }
                            sm.L_rs[e - e0] = rs;
                            sm.L_d[e - e0] = dn.x;
                            sm.L_ph[e - e0] = jb;
                            if (nb > 1) {
                                const unsigned br = 1u << (rs.x & 31), bs = 1u << (rs.y & 31);
                                const unsigned o1 = atomicOr(sm.bm + (rs.x >> 5), br);
                                const unsigned o2 = atomicOr(sm.bm + (rs.y >> 5), bs);
                                if ((o1 & br) | (o2 & bs)) s_conflict = 1;
                            }
                        }
                        bar_apply();
                        const int conflict = s_conflict;
                        if (!conflict) {
                            apply_rows(sm.L_rs, sm.L_d, sm.L_ph, -1, 0, e1 - e0, w2, Wb, Tb, ta);
                        } else {
                            for (int jb = 0; jb < nb; ++jb) {
                                const int lo = max(sm.s_off[jb * nsh], e0) - e0;
                                const int hi = min(sm.s_off[(jb + 1) * nsh], e1) - e0;
                                if (lo < hi) apply_rows(sm.L_rs, sm.L_d, sm.L_ph, -1, lo, hi, w2, Wb, Tb, ta);
                                bar_apply();
                            }
                        }
                        bar_apply();
                        if (nb > 1) {
                            for (int e = ta; e < e1 - e0; e += kApply) {
                                const int2 rs = sm.L_rs[e];
                                atomicAnd(sm.bm + (rs.x >> 5), ~(1u << (rs.x & 31)));
                                atomicAnd(sm.bm + (rs.y >> 5), ~(1u << (rs.y & 31)));
                            }
                        }
                        bar_apply();
                        if (ta == 0) s_conflict = 0;
                    }
                }
                C = k1;
                cph = ph0 + (k1 - k0);
                cit = it0;
                ++nbatch;
            }
            t_busy += PCLK() - t0;
            if (stopg >= 0 && C >= stopg) break;
        }
        if (prof && ta == 0) {
            prof[4] = (unsigned long long)t_busy;
            prof[5] = (unsigned long long)t_idle;
            prof[6] = (unsigned long long)nbatch;
            prof[10] = (unsigned long long)t_head;
            prof[11] = (unsigned long long)t_diag;
            prof[12] = (unsigned long long)t_h0;
            prof[13] = (unsigned long long)t_h1;
            prof[14] = (unsigned long long)t_h2;
        }
    }
    __syncthreads();
    if (bl == 0 && tid == 0) {
        a.status[0] = s_iters;
        a.status[1] = s_conv;
    }
}
#undef PCLK


// --------------------------------------------------------------- layout kernels
// Slab storage: local slab b (global column block blk0 + b), row i, column j of the slab at
// b * ss + i * rs + j -- slab layout ss = p*w, rs = w; row-major layout ss = w, rs = nblk*w.

// Row-major p x p (leading dim ld) -> nblk slabs of width w starting at global
// column block blk0 (zero padding past column p).
__global__ void pack_slabs_kernel(const double* __restrict__ src, long long ld, double* __restrict__ dst,
                                  int p, int w, long long ss, long long rs, int nblk, int blk0) {
    const long long total = (long long)nblk * p * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / ((long long)p * w);
        const long long rem = e - b * p * w;
        const int i = (int)(rem / w);
        const int j = (int)(rem - (long long)i * w);
        const long long c = (blk0 + b) * w + j;
        dst[b * ss + (long long)i * rs + j] = (c < p) ? src[(long long)i * ld + c] : 0.0;
    }
}

// Slabs -> row-major p x ncols (ncols = columns the slabs hold, clipped to p).
__global__ void unpack_slabs_kernel(const double* __restrict__ src, double* __restrict__ dst, int p, int w,
                                    long long ss, long long rs, int ncols) {
    const long long total = (long long)p * ncols;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / ncols);
        const int c = (int)(e - (long long)i * ncols);
        const int b = c / w;
        dst[e] = src[(long long)b * ss + (long long)i * rs + (c - b * w)];
    }
}

__global__ void rowmajor_diag_kernel(const double* __restrict__ src, double* __restrict__ diag, int p) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x)
        diag[i] = src[(long long)i * p + i];
}

__global__ void slab_set_identity_kernel(double* __restrict__ slab, int p, int w, long long ss, long long rs, int nblk,
                                         int blk0) {
    const int c0 = blk0 * w;
    const int c1 = min(p, (blk0 + nblk) * w);
    for (int c = c0 + blockIdx.x * blockDim.x + threadIdx.x; c < c1; c += gridDim.x * blockDim.x) {
        const int b = c / w - blk0;
        slab[(long long)b * ss + (long long)c * rs + (c - (b + blk0) * w)] = 1.0;
    }
}

// Count exact non-zeros of the strict upper triangle (model.py:249-253).
__global__ void slab_edge_count_kernel(const double* __restrict__ slab, int p, int w, long long ss, long long rs,
                                       int nblk, int blk0, unsigned long long* __restrict__ out) {
    unsigned long long local = 0;
    const long long total = (long long)nblk * p * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / ((long long)p * w);
        const long long rem = e - b * p * w;
        const int i = (int)(rem / w);
        const long long j = rem - (long long)i * w;
        const long long c = (blk0 + b) * w + j;
        if (c < p && i < c && slab[b * ss + (long long)i * rs + j] != 0.0) ++local;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

// W (slab) = Omega_init * T for a warm start, from a CSR copy of Omega_init.
// Row i of W is sum_k om[i,k] T[k,:]; each block streams its own slab.
__global__ void wform_init_csr_kernel(const long long* __restrict__ rowptr, const int* __restrict__ colidx,
                                      const double* __restrict__ vals, const double* __restrict__ Tslab,
                                      double* __restrict__ Wslab, int p, int w, long long ss, long long rs) {
    const int b = blockIdx.y;
    const double* Tb = Tslab + (long long)b * ss;
    double* Wb = Wslab + (long long)b * ss;
    const int w2 = w >> 1;
    const long long items = (long long)p * w2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < items;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / w2);
        const int j2 = (int)(idx - (long long)i * w2);
        double2 acc = make_double2(0.0, 0.0);
        for (long long e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const double v = vals[e];
            const double2 tv = __ldg(reinterpret_cast<const double2*>(Tb + (long long)colidx[e] * rs) + j2);
            acc.x = fma(v, tv.x, acc.x);
            acc.y = fma(v, tv.y, acc.y);
        }
        reinterpret_cast<double2*>(Wb + (long long)i * rs)[j2] = acc;
    }
}


// ------------------------------------------------------------------ launchers
int wform_tdiag_in_smem(int p) { return p <= 12288; }

int wform_lag_cap(int w, int m) {
    int l = WFORM_MAX_LAG < m ? WFORM_MAX_LAG : m;
    while (l > 1 && (size_t)kSlots * (2 + l) * w * sizeof(double) > 150 * 1024) --l;
    return l;
}

size_t wform_smem_bytes(int w, int p, int nblk, int lmax) {
    size_t b = sizeof(double) * (size_t)kSlots * (2 + lmax) * w;
    b += (sizeof(int2) + 2 * sizeof(double) + sizeof(int)) * kPairCap;
    b += sizeof(int) * ((size_t)kBatch * nblk + 1);
    b = (b + 15) & ~(size_t)15;
    b += sizeof(unsigned) * (size_t)((p + 31) / 32);
    b = (b + 15) & ~(size_t)15;
    if (wform_tdiag_in_smem(p)) b += sizeof(double) * (size_t)p;
    return b;
}

cudaError_t launch_pcd_wform(const WformArgs& args, int nblk, cudaStream_t st) {
    const size_t smem = wform_smem_bytes(args.w, args.p, args.nblk_tot, args.lmax);
    const void* fn = args.prof ? (const void*)pcd_wform_kernel<true> : (const void*)pcd_wform_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    WformArgs copy = args;
    void* kargs[] = {&copy};
    return cudaLaunchCooperativeKernel(fn, dim3(nblk), dim3(kThreads), kargs, smem, st);
}

cudaError_t wform_max_blocks(int w, int p, int nblk_tot, int* max_blocks) {
    const size_t smem = wform_smem_bytes(w, p, nblk_tot, wform_lag_cap(w, p + (p & 1) - 1));
    if (smem > 227 * 1024) {
        *max_blocks = 0;
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(pcd_wform_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(pcd_wform_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcd_wform_kernel<false>, kThreads, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    *max_blocks = per_sm * nsm;
    return cudaSuccess;
}

static int grid_for(long long total) {
    long long g = (total + 255) / 256;
    if (g > 148LL * 16) g = 148LL * 16;
    if (g < 1) g = 1;
    return (int)g;
}

cudaError_t launch_pack_slabs(const double* src, long long ld, double* dst, int p, int w, long long ss, long long rs,
                              int nblk, int blk0, cudaStream_t st) {
    pack_slabs_kernel<<<grid_for((long long)nblk * p * w), 256, 0, st>>>(src, ld, dst, p, w, ss, rs, nblk, blk0);
    return cudaGetLastError();
}

cudaError_t launch_unpack_slabs(const double* src, double* dst, int p, int w, long long ss, long long rs, int nblk,
                                int blk0, cudaStream_t st) {
    const int ncols = max(0, min(p, (blk0 + nblk) * w) - blk0 * w);
    unpack_slabs_kernel<<<grid_for((long long)p * ncols), 256, 0, st>>>(src, dst, p, w, ss, rs, ncols);
    return cudaGetLastError();
}

cudaError_t launch_rowmajor_diag(const double* src, double* diag, int p, cudaStream_t st) {
    rowmajor_diag_kernel<<<grid_for(p), 256, 0, st>>>(src, diag, p);
    return cudaGetLastError();
}

cudaError_t launch_slab_identity(double* slab, int p, int w, long long ss, long long rs, int nblk, int blk0,
                                 cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(slab, 0, sizeof(double) * (size_t)nblk * p * w, st);
    if (e != cudaSuccess) return e;
    slab_set_identity_kernel<<<grid_for((long long)nblk * w), 256, 0, st>>>(slab, p, w, ss, rs, nblk, blk0);
    return cudaGetLastError();
}

cudaError_t launch_slab_edge_count(const double* slab, int p, int w, long long ss, long long rs, int nblk, int blk0,
                                   unsigned long long* out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    slab_edge_count_kernel<<<grid_for((long long)nblk * p * w), 256, 0, st>>>(slab, p, w, ss, rs, nblk, blk0, out);
    return cudaGetLastError();
}

cudaError_t launch_wform_init_csr(const long long* rowptr, const int* colidx, const double* vals, const double* Tslab,
                                  double* Wslab, int p, int w, long long ss, long long rs, int nblk, cudaStream_t st) {
    long long items = (long long)p * (w >> 1);
    int gx = (int)((items + 255) / 256);
    if (gx > 64) gx = 64;
    wform_init_csr_kernel<<<dim3(gx, nblk), 256, 0, st>>>(rowptr, colidx, vals, Tslab, Wslab, p, w, ss, rs);
    return cudaGetLastError();
}

}  // namespace concord
