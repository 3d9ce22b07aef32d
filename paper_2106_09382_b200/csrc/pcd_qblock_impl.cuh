// CONCORD-PCD fit kernel with TEMPORAL BLOCKING of the colour chain in pair
// space (sm_100a).  Same algorithm, arithmetic and results as pcd_wform.cu --
// bitwise -- with D colour phases per grid barrier instead of one.
//
// The circle schedule (schedule.py:68-88) moves every id one position per
// round, so the pair index q of any row changes by at most one per colour
// (q = 0 and q = half-1 reflect), and the two rows of a pair share it.  Hence
// pair q of colour k+1 depends only on pairs q-1, q, q+1 of colour k through
// the rows it shares with them: a 1-D stencil in q.  A CTA that owns the
// pairs [q_lo, q_hi) can therefore evaluate D consecutive colours after ONE
// grid barrier by also evaluating, redundantly, a halo of D-1-d pairs on each
// side at colour d of the block (identical arithmetic in every CTA that
// evaluates a pair, so the halo copies agree bit for bit).
//
// Per block of D phases (blocks never straddle a sweep; the diagonal phase
// closes the sweep's last block):
//  * chain warps.  The cells W[x,c] / Om[x,c] the block's pairs (and halo) need
//    come from the STAGE, written in global memory by the slab owners with
//    watermark C'(B) = (start of block B-3) - 1.  Part A of a block's cells --
//    stage values, in-block T entries, pair slots, the deltas of blocks B-3 and
//    B-2 (per-row delta ring; T entries only where a delta is non-zero) -- is
//    built by the chain warps the colours leave free (the prefetch group) while
//    block B-1's colours run, into the second of two cell buffers.  After the
//    barrier, part B folds in block B-1's deltas; then the colours run one after
//    another in shared memory with the block's own deltas; one pass publishes
//    the own pairs' delta ring and non-zero delta lists; the diagonal phase
//    writes the (delta, new) vector.  One arrive per block, once the block after
//    next is staged.
//  * apply warps (as pcd_wform.cu): stream the delta lists into the own slab in
//    phase order through a per-thread cp.async ring (per-row chains where a
//    batch moves a row more than once), run the dense diagonal step, and stage
//    the cells of upcoming blocks, bringing them forward from their own
//    watermark with exactly the FMAs they will apply to the slab.
//
// Every published value is thus the value of the sequential W-form (same
// FMAs, same order), and the results equal pcd_wform.cu's bit for bit.
// Shared-memory plan (cell buffers, T diagonal, ring depth) per p: capi.cu.
// Implementation of the blocked kernel, compiled once per chain-warp variant: the including
// translation unit defines QB_NS, QB_NS_CHAIN_WARPS and the setmaxnreg budgets QB_NS_REGS_CHAIN /
// QB_NS_REGS_APPLY (0: no register redistribution).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "pcd_wform.h"

namespace concord {
namespace QB_NS {

constexpr int kThreads = WFORM_THREADS;
constexpr int kChainWarps = QB_NS_CHAIN_WARPS;
constexpr int kChain = kChainWarps * 32;
constexpr int kApply = kThreads - kChain;
constexpr int kApplyWarps = kApply / 32;
constexpr int kPairCap = WFORM_PAIR_CAP;
constexpr int kBatch = WFORM_BATCH;
constexpr int kUnroll = 2;
constexpr int kDMax = QB_DMAX;
constexpr int kChainN = 32;   // batches with row conflicts up to this many entries: per-row chains
#ifndef QB_POLL_NS
#define QB_POLL_NS 20         // back-off of the chain's spin loops (barrier, own stager)
#endif
#ifndef QB_IDLE_NS
#define QB_IDLE_NS 32         // back-off of the idle apply warps
#endif

__device__ __forceinline__ void bar_chain() { asm volatile("bar.sync 1, %0;" ::"n"(kChain) : "memory"); }
__device__ __forceinline__ void bar_apply() { asm volatile("bar.sync 2, %0;" ::"n"(kApply) : "memory"); }
__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_vol(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}

// Clock read that cannot issue before `dep` is available (profiling only).
__device__ __forceinline__ long long clock_after(double dep) {
    long long t;
    asm volatile(
        "{\n .reg .pred pp;\n setp.eq.f64 pp, %1, 0d7FF0000000000001;\n @pp mov.u64 %0, 0;\n"
        " @!pp mov.u64 %0, %%clock64;\n}"
        : "=l"(t)
        : "d"(dep)
        : "memory");
    return t;
}

// Partners of row x along consecutive phases (in-sweep phase ph = 0..m, m = the
// diagonal, where the "partner" is x itself), division-free after the first:
// circle_partner(x, k) - 1 = (3m - x - 1 - 2k) mod m steps by -2 per colour (-1 for
// id 0), and the diagonal phase does not advance k (k = m is k = 0 mod m).
struct PartnerWalk {
    int x, m, v, ph;
    __device__ __forceinline__ PartnerWalk(int x_, int ph_, int m_) : x(x_), m(m_), ph(ph_) {
        const int k = (ph_ == m_) ? 0 : ph_;
        // division-free: m-1-k is in [0, m), 3m-x-1-2k in [1, 3m-2] (0 <= k < m, 1 <= x <= m)
        if (x_ == 0) {
            v = m_ - 1 - k;
        } else {
            v = 3 * m_ - x_ - 1 - 2 * k;
            v -= (v >= 2 * m_) ? 2 * m_ : ((v >= m_) ? m_ : 0);
        }
    }
    __device__ __forceinline__ int y() const {
        if (ph == m) return x;
        return (x != 0 && 1 + v == x) ? 0 : 1 + v;
    }
    __device__ __forceinline__ void next() {
        if (ph == m) {
            ph = 0;
        } else {
            ++ph;
            v -= (x == 0) ? 1 : 2;
            if (v < 0) v += m;
        }
    }
};

// ld.global.cg of a double when `on`, else 0.0, without a branch.
__device__ __forceinline__ double ldcg_if(const double* ptr, bool on) {
    double v;
    asm volatile(
        "{\n .reg .pred pp;\n setp.ne.b32 pp, %2, 0;\n mov.f64 %0, 0d0000000000000000;\n"
        " @pp ld.global.cg.f64 %0, [%1];\n}"
        : "=d"(v)
        : "l"(ptr), "r"((int)on));
    return v;
}

// Geometry of global block b: first global phase g0, its phase-in-sweep ph0, length len.
struct Blk {
    int g0, ph0, len, sweep;
};
// b / NB without a division (Granlund-Montgomery; nb_magic / nb_shift precomputed by the host)
__device__ __forceinline__ int div_nb(int b, unsigned magic, int shift) {
    if (shift < 0) return b;  // NB == 1
    const unsigned t = __umulhi((unsigned)b, magic);
    return (int)((t + (((unsigned)b - t) >> 1)) >> shift);
}
__device__ __forceinline__ Blk block_at(int b, int m, int D, int NB, unsigned magic, int shift) {
    Blk k;
    k.sweep = div_nb(b, magic, shift);
    const int j = b - k.sweep * NB;
    k.ph0 = j * D;
    k.len = min(D, m + 1 - k.ph0);
    k.g0 = k.sweep * (m + 1) + k.ph0;
    return k;
}
// Watermark of the stage of block b: every phase <= C' is already in the staged cells.
// C'(b) = start of block b-3, minus one: the deltas it needs are known once the chain is at
// block b-3, so the stager has a block of slack before the chain needs it (at block b-2).
__device__ __forceinline__ int stage_mark(int b, int m, int D, int NB, unsigned magic, int shift) {
    return (b < 3) ? -1 : block_at(b - 3, m, D, NB, magic, shift).g0 - 1;
}

// Chain warps the colours of a block need: one thread per pair of the widest colour.
__host__ __device__ __forceinline__ int colour_warps(int share, int D) {
    const int n = (share + 2 * (D - 1) + 31) / 32;
    return n < kChainWarps ? n : kChainWarps;
}

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

// Row streams of delta-list entries [e_lo, e_hi) (shared-memory indices; only batch phase
// `only` when only >= 0): W[dst, own] = fma(d, T[src, own], W[dst, own]) for both rows of every
// pair, with the loads off the register file: every apply
// thread keeps S items in flight through its own ring of
// shared-memory slots (cp.async, 32 B per item: the W and T chunk), so an SM
// holds kApply * S * 32 B of row traffic in flight instead of the few double2 pairs the
// registers allow. Each thread only reads the
// slots it filled, so no barrier is needed; cp.async.wait_group orders them.
__device__ __forceinline__ void apply_rows_async(const int2* L_rs, const double* L_d, const int* L_ph, int only,
                                                 int e_lo, int e_hi, int w2, unsigned per_magic, int per_shift,
                                                 long long ld2, double* __restrict__ Wb,
                                                 const double* __restrict__ Tb, double2* ring, int ta, int S) {
    const int per = 2 * w2;
    const int items = (e_hi - e_lo) * per;
    const int nmine = items > ta ? (items - ta + kApply - 1) / kApply : 0;
    // item idx = ta + i * kApply -> (entry q, position rem in the entry), stepped without division
    // x / per as a multiply-shift (per = w; host-computed magic): no division per pass
    const int dq = div_nb(kApply, per_magic, per_shift), dr = kApply - dq * per;
    struct Cursor {
        int q, rem;
    };
    auto step = [&](Cursor& c) {
        c.q += dq;
        c.rem += dr;
        if (c.rem >= per) {
            c.rem -= per;
            ++c.q;
        }
    };
    auto locate = [&](const Cursor& c, int& e, int& off_w, int& off_t) {
        e = e_lo + c.q;
        const int h = c.rem >= w2;
        const int j2 = c.rem - h * w2;
        const int2 rs = L_rs[e];
        off_w = (h ? rs.y : rs.x) * ld2 + j2;
        off_t = (h ? rs.x : rs.y) * ld2 + j2;
    };
    const int tq = div_nb(ta, per_magic, per_shift);
    Cursor ci{tq, ta - tq * per};  // next item to issue
    Cursor cc = ci;                               // next item to complete
    int si = 0, sc = 0;  // ring slots of the next issue / the next completion
    auto issue = [&]() {
        int e, ow, ot;
        locate(ci, e, ow, ot);
        if (only < 0 || L_ph[e] == only) {
            double2* slot = ring + (size_t)(si * 2) * kApply + ta;
            const unsigned sw = (unsigned)__cvta_generic_to_shared(slot);
            const unsigned st = (unsigned)__cvta_generic_to_shared(slot + kApply);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sw),
                         "l"(reinterpret_cast<const double2*>(Wb) + ow)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st),
                         "l"(reinterpret_cast<const double2*>(Tb) + ot)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        si = (si + 1 == S) ? 0 : si + 1;
        step(ci);
    };
    // prologue: S - 1 items in flight; then one issue per completed item, and in the
    // tail (nothing left to issue) wait for everything.  S is 2, 4, 6 or 8 (shared-memory budget).
    int ni = min(nmine, S - 1);
    for (int i = 0; i < ni; ++i) issue();
    for (int j = 0; j < nmine; ++j) {
        if (ni < nmine) {
            issue();
            ++ni;
            if (S == 8) asm volatile("cp.async.wait_group 7;" ::: "memory");
            else if (S == 6) asm volatile("cp.async.wait_group 5;" ::: "memory");
            else if (S == 4) asm volatile("cp.async.wait_group 3;" ::: "memory");
            else asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        int e, ow, ot;
        locate(cc, e, ow, ot);
        if (only < 0 || L_ph[e] == only) {
            const double2* slot = ring + (size_t)(sc * 2) * kApply + ta;
            double2 wv = slot[0];
            const double2 tv = slot[kApply];
            const double d = L_d[e];
            wv.x = fma(d, tv.x, wv.x);
            wv.y = fma(d, tv.y, wv.y);
            reinterpret_cast<double2*>(Wb)[ow] = wv;
        }
        sc = (sc + 1 == S) ? 0 : sc + 1;
        step(cc);
    }
}


// Rows of a batch whose phases move some row more than once (entries [0, nent), all in
// shared memory, phase L_ph).  Every half-entry (dst row, src row, delta) is linked to the
// next half-entry of the batch with the same dst row (phase order); the first of each chain
// loads W[dst, chunk] once, the T chunks of the whole chain at once, and applies the FMAs in
// phase order -- the same operations, in the same order, as phase-by-phase passes, in one
// round trip instead of one per phase.
__device__ __noinline__ void apply_chains(const int2* L_rs, const double* L_d, const int* L_ph, int nent, int w2,
                                          unsigned w2_magic, int w2_shift,
                                             int ld2, double* __restrict__ Wb, const double* __restrict__ Tb, short* s_next,
                                             unsigned char* s_first, int ta) {
    for (int he = ta; he < 2 * nent; he += kApply) {
        const int e = he >> 1;
        const int2 rs = L_rs[e];
        const int dst = (he & 1) ? rs.y : rs.x;
        const int ph = L_ph[e];
        int nxt = -1, nph = 0x7fffffff;
        bool first = true;
        for (int e2 = 0; e2 < nent; ++e2) {
            const int2 r2 = L_rs[e2];
            const int ph2 = L_ph[e2];
            if (r2.x == dst || r2.y == dst) {
                if (ph2 < ph) first = false;
                else if (ph2 > ph && ph2 < nph) {
                    nph = ph2;
                    nxt = 2 * e2 + (r2.y == dst ? 1 : 0);
                }
            }
        }
        s_next[he] = (short)nxt;
        s_first[he] = first ? 1 : 0;
    }
    bar_apply();
    const int items = 2 * nent * w2;
    // item idx = (half-entry he, chunk j2), stepped without division
    const int sq = div_nb(kApply, w2_magic, w2_shift), sr = kApply - sq * w2;
    int che = div_nb(ta, w2_magic, w2_shift), cj2 = ta - che * w2;
    for (int idx = ta; idx < items; idx += kApply) {
        const int he = che, j2 = cj2;
        che += sq;
        cj2 += sr;
        if (cj2 >= w2) {
            cj2 -= w2;
            ++che;
        }
        if (!s_first[he]) continue;
        const int2 rs0 = L_rs[he >> 1];
        const int dst = (he & 1) ? rs0.y : rs0.x;
        double2* wp = reinterpret_cast<double2*>(Wb) + (long long)dst * ld2 + j2;
        double2 wv = __ldcg(wp);
        // the chain, four links at a time: T loads of a group back to back, then its FMAs
        int k = he;
        while (k >= 0) {
            int srcs[4];
            double ds[4];
            int len = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k >= 0) {
                    const int2 r = L_rs[k >> 1];
                    srcs[u] = (k & 1) ? r.x : r.y;
                    ds[u] = L_d[k >> 1];
                    len = u + 1;
                    k = s_next[k];
                }
            }
            double2 tv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < len) tv[u] = __ldcg(reinterpret_cast<const double2*>(Tb) + (long long)srcs[u] * ld2 + j2);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < len) {
                    wv.x = fma(ds[u], tv[u].x, wv.x);
                    wv.y = fma(ds[u], tv[u].y, wv.y);
                }
        }
        *wp = wv;
    }
}

#define ROWS(Lrs, Ld, Lph, only, lo, hi, w2_, Wb_, Tb_, ring_, ta_) \
    apply_rows_async(Lrs, Ld, Lph, only, lo, hi, w2_, a.w_magic, a.w_shift, ld2, Wb_, Tb_, ring_, ta_, a.ring_stages)

#define QB_COPIES_RT(r) _Pragma("unroll") for (int r = 0; r < WFORM_MAX_SHARDS; ++r) if (r < a.G)
// In the kernel: one copy unless the launch is sharded (kShard), so the unsharded instance carries
// no per-copy predicates in its store loops.
#define QB_COPIES(r) _Pragma("unroll") for (int r = 0; r < (kShard ? WFORM_MAX_SHARDS : 1); ++r) if (!kShard || r < a.G)

// Arrive on the grid barrier of every shard: this CTA's exchange-buffer stores (its own and, through
// the CTA barrier before the call, its other threads') become visible at GPU scope -- or system
// scope when the shards are separate GPUs reached over NVLink -- then every copy of the counter
// is bumped.  One GPU, one copy: a release reduction (no separate fence).
__device__ __forceinline__ void qb_arrive(const QbArgs& a) {
    if (a.sys_scope) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        QB_COPIES_RT(r) asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(a.x.bar[r]) : "memory");
    } else if (a.G == 1) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.x.bar[0]) : "memory");
    } else {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        QB_COPIES_RT(r) asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(a.x.bar[r]) : "memory");
    }
}

__device__ __forceinline__ void wait_counter(const unsigned long long* ctr, unsigned long long target, int blk,
                                             long long* hang, int sys) {
    unsigned long long v;
    const unsigned long long t0 = globaltimer_ns();
    int spins = 0;
    do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (QB_POLL_NS && v < target) __nanosleep(QB_POLL_NS);  // leave issue slots to this SMSP's apply warps
        if (++spins == 4096) {
            spins = 0;
            if (globaltimer_ns() - t0 > kHangNs) hang_report(hang, 0, blk, (long long)v, (long long)target, 0, 0);
        }
    } while (v < target);
    if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

struct Layout {
    int lo[kDMax], cb[kDMax + 1], slot[kDMax + 1], rdc[kDMax], lsl[kDMax];
    int ncell, rd0, ph0w, rdb, phb;
};

// Dynamic shared memory of the blocked kernel, addressed by 32-bit offsets from one
// shared base (one register per array, native shared addressing) instead of generic pointers.
extern __shared__ __align__(16) unsigned char qb_smem[];

struct Smem {
    unsigned o_L_rs;  // [kPairCap]  delta-list chunk
    unsigned o_L_d;  // [kPairCap]
    unsigned o_L_new;  // [kPairCap]
    unsigned o_L_ph;  // [kPairCap]
    unsigned o_s_off;  // [kBatch * nblk + 1]
    unsigned o_bm;  // [(p + 31) / 32]
    unsigned o_td;  // [p] T diagonal, or NULL
    unsigned o_cX;  // [cellcap] row of each block cell (-1: phantom)
    unsigned o_cC;  // [cellcap] column of each block cell
    unsigned o_cW;  // [cellcap] cell value brought forward to the start of the block
    unsigned o_cO;  // [cellcap] Omega of the cell
    unsigned o_cT;  // [nbuf][cellcap][D-1] T entries of the block's earlier phases
    unsigned o_sd;  // [kDMax][rmax] delta of each pair of the block's phases (extended ranges)
    unsigned o_cQ;  // [nbuf][cellcap][D-1] index into sd[i] of the cell row's pair at in-block phase i
    unsigned o_snv;  // [kDMax][share] new value of each own pair of the block's colours
    unsigned o_hd_rs;  // [kBatch * nblk] first entry of each list segment of a batch
    unsigned o_hd_dn;  // [kBatch * nblk]
    unsigned o_ring;  // [ring_stages][2][kApply] per-thread cp.async slots of the row streams
    __device__ __forceinline__ int2* L_rs() const { return reinterpret_cast<int2*>(qb_smem + o_L_rs); }
    __device__ __forceinline__ double* L_d() const { return reinterpret_cast<double*>(qb_smem + o_L_d); }
    __device__ __forceinline__ double* L_new() const { return reinterpret_cast<double*>(qb_smem + o_L_new); }
    __device__ __forceinline__ int* L_ph() const { return reinterpret_cast<int*>(qb_smem + o_L_ph); }
    __device__ __forceinline__ int* s_off() const { return reinterpret_cast<int*>(qb_smem + o_s_off); }
    __device__ __forceinline__ unsigned* bm() const { return reinterpret_cast<unsigned*>(qb_smem + o_bm); }
    __device__ __forceinline__ double* td() const { return reinterpret_cast<double*>(qb_smem + o_td); }
    __device__ __forceinline__ int* cX() const { return reinterpret_cast<int*>(qb_smem + o_cX); }
    __device__ __forceinline__ int* cC() const { return reinterpret_cast<int*>(qb_smem + o_cC); }
    __device__ __forceinline__ double* cW() const { return reinterpret_cast<double*>(qb_smem + o_cW); }
    __device__ __forceinline__ double* cO() const { return reinterpret_cast<double*>(qb_smem + o_cO); }
    __device__ __forceinline__ double* cT() const { return reinterpret_cast<double*>(qb_smem + o_cT); }
    __device__ __forceinline__ double* sd() const { return reinterpret_cast<double*>(qb_smem + o_sd); }
    __device__ __forceinline__ short* cQ() const { return reinterpret_cast<short*>(qb_smem + o_cQ); }
    __device__ __forceinline__ double* snv() const { return reinterpret_cast<double*>(qb_smem + o_snv); }
    __device__ __forceinline__ int2* hd_rs() const { return reinterpret_cast<int2*>(qb_smem + o_hd_rs); }
    __device__ __forceinline__ double2* hd_dn() const { return reinterpret_cast<double2*>(qb_smem + o_hd_dn); }
    __device__ __forceinline__ double2* ring() const { return reinterpret_cast<double2*>(qb_smem + o_ring); }
};

// kProf: the phase profiler (CONCORD_PHASE_PROFILE); the production instantiation carries
// no timers at all (they would hold ~30 registers across the loops).
template <bool kProf, bool kShard>
#define PCLK() (kProf ? clock64() : 0ll)
__global__ void __launch_bounds__(kThreads, 1) pcd_qblock_kernel(QbArgs a) {
    __shared__ int s_epoch, s_blk, s_stop, s_staged, s_iters, s_conv;
    __shared__ int s_cnt[kDMax];
    __shared__ short s_next[2 * kChainN];
    __shared__ unsigned char s_first[2 * kChainN];
    __shared__ int s_aE, s_aBlk, s_aStop, s_nent, s_multi, s_conflict;
    __shared__ int s_wsum[kApplyWarps];
    __shared__ Layout s_ly[2];
    __shared__ double s_red[4][kApplyWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bl = blockIdx.x;       // slab of this launch
    const int b = a.blk0 + bl;       // global CTA = global column block (pairs, list segments)
    const int nblk = a.nblk_tot;     // CTAs over all shards
    const int shard = b / a.nblk_loc;  // whose copy of the exchange buffers this CTA reads
    const int p = a.p, m = a.m, w = a.w, w2 = a.w >> 1, half = a.half;
    const int D = a.D, NB = a.NB;
    const int dm1 = D - 1;  // stride of the per-cell arrays cT, cQ
    const int c0 = b * w;
    const int wl = max(0, min(w, p - c0));
    const int q_lo = min(b * a.share, half), q_hi = min(q_lo + a.share, half);
    // slab bl of this launch: element (row x, column c0 + j) at base + bl * a.slab + x * ld + j
    // (row-major layout: a.slab = w, ld = the launch's columns; slab layout: a.slab = p * w, ld = w)
    const int ld = a.ld, ld2 = a.ld >> 1;
    double* __restrict__ Wb = a.W + (long long)bl * a.slab;
    const double* __restrict__ Tb = a.T + (long long)bl * a.slab;
    double* __restrict__ Ob = a.Om + (long long)bl * a.slab;
    // this shard's copies (read side); every write goes to all copies (QB_COPIES)
    const int* lcntL = a.x.list_cnt[0];
    const int2* lrsL = a.x.list_rs[0];
    const double2* ldnL = a.x.list_dn[0];
    const double* stWL = a.x.stW[0];
    const double* stOL = a.x.stO[0];
    const double* stTL = a.x.stT[0];
    const double* dringL = a.x.dring[0];
    const double2* diagvL = a.x.diagv[0];
    const unsigned long long* barL = a.x.bar[0];
    const unsigned long long* dmaxL = a.x.dmax[0];
#pragma unroll
    for (int r = 1; r < (kShard ? WFORM_MAX_SHARDS : 1); ++r)
        if (r == shard) {
            lcntL = a.x.list_cnt[r];
            lrsL = a.x.list_rs[r];
            ldnL = a.x.list_dn[r];
            stWL = a.x.stW[r];
            stOL = a.x.stO[r];
            stTL = a.x.stT[r];
            dringL = a.x.dring[r];
            diagvL = a.x.diagv[r];
            barL = a.x.bar[r];
            dmaxL = a.x.dmax[r];
        }

    Smem sm;
    {
        unsigned off = 0;
        auto take = [&](size_t bytes) {
            const unsigned r = off;
            off += (unsigned)((bytes + 15) & ~(size_t)15);
            return r;
        };
        sm.o_L_rs = take(sizeof(int2) * kPairCap);
        sm.o_L_d = take(sizeof(double) * kPairCap);
        sm.o_L_new = take(sizeof(double) * kPairCap);
        sm.o_L_ph = take(sizeof(int) * kPairCap);
        sm.o_s_off = take(sizeof(int) * ((size_t)kBatch * nblk + 1));
        sm.o_bm = take(sizeof(unsigned) * (size_t)((p + 31) / 32));
        sm.o_cX = take(sizeof(int) * a.nbuf * (size_t)a.cellcap);
        sm.o_cC = take(sizeof(int) * a.nbuf * (size_t)a.cellcap);
        sm.o_cW = take(sizeof(double) * a.nbuf * (size_t)a.cellcap);
        sm.o_cO = take(sizeof(double) * a.nbuf * (size_t)a.cellcap);
        sm.o_cT = take(sizeof(double) * a.nbuf * (size_t)a.cellcap * dm1);
        sm.o_sd = take(sizeof(double) * (size_t)kDMax * a.rmax);
        sm.o_cQ = take(sizeof(short) * a.nbuf * (size_t)a.cellcap * dm1);
        sm.o_snv = take(sizeof(double) * (size_t)kDMax * a.share);
        sm.o_hd_rs = take(sizeof(int2) * (size_t)kBatch * nblk);
        sm.o_hd_dn = take(sizeof(double2) * (size_t)kBatch * nblk);
        sm.o_ring = take(sizeof(double2) * 2 * (size_t)kApply * a.ring_stages);
        sm.o_td = a.tdiag_smem ? take(sizeof(double) * (size_t)p) : 0xffffffffu;
    }
    if (a.tdiag_smem)
        for (int i = tid; i < p; i += kThreads) sm.td()[i] = __ldg(a.tdiag + i);
    for (int i = tid; i < (p + 31) / 32; i += kThreads) sm.bm()[i] = 0u;
#define TD(i) (a.tdiag_smem ? sm.td()[i] : __ldg(a.tdiag + (i)))

    // ---- stage blocks 0 and 1 from the initial W, Omega (watermark -1)
    for (int bb = 0; bb < 2 && bb < 2 * NB; ++bb) {
        const Blk k = block_at(bb, m, D, NB, a.nb_magic, a.nb_shift);
        for (int idx = tid; idx < k.len * wl; idx += kThreads) {
            const int i = idx / wl, j = idx - i * wl;
            const int Q = k.g0 + i;
            const int c = c0 + j;
            const int x = pub_row(k.ph0 + i, c, m, p);
            if (x < 0) continue;
            const size_t so = (size_t)(Q % a.sr) * p + c;
            const double wv0 = Wb[(long long)x * ld + j], ov0 = Ob[(long long)x * ld + j];
            QB_COPIES(r) {
                a.x.stW[r][so] = wv0;
                a.x.stO[r][so] = ov0;
            }
            for (int ii = 0; ii < i; ++ii) {
                const int y = src_row(k.ph0 + ii, x, m);
                const double tv0 = (y < p) ? Tb[(long long)y * ld + j] : 0.0;
                QB_COPIES(r) a.x.stT[r][((size_t)(Q % a.sr) * (kDMax - 1) + ii) * p + c] = tv0;
            }
        }
    }
    if (tid == 0) {
        s_epoch = -1;
        s_blk = -1;
        s_stop = -1;
        s_staged = 1;
        for (int d = 0; d < kDMax; ++d) s_cnt[d] = 0;
        s_conflict = 0;
    }
    __syncthreads();

    unsigned long long* prof = (kProf && a.prof && bl == 0) ? a.prof : nullptr;

    if (warp < kChainWarps) {
#if QB_NS_REGS_CHAIN
        // warp-group register split (chain and apply roles aligned to warp groups): the chain
        // warps hand registers to the apply warps
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(QB_NS_REGS_CHAIN));
#endif
        // ================================================================ chain warps
        const int tc = tid;
        // The colours of a block need one thread per pair of the widest colour (own pairs plus
        // halo): the last ncw chain warps (the colour group).  The other chain warps (the
        // prefetch group) meanwhile build part A of the next block's cells, so only part B
        // (the previous block's deltas) is left between a barrier and the colours.  When the
        // colours need every chain warp, part A runs after the arrive instead.
        // colour_warps_min < 0: exactly -colour_warps_min warps (tuning; the colours loop over pairs)
        const int ncw0 = (a.colour_warps_min < 0) ? min(-a.colour_warps_min, kChainWarps)
                                                  : max(colour_warps(a.share, D), min(a.colour_warps_min, kChainWarps));
        const bool overlap = ncw0 < kChainWarps && a.nbuf == 2;
        const int ncw = overlap ? ncw0 : kChainWarps;
        const int cg0 = kChain - 32 * ncw;  // first thread of the colour group
        const int ng = 32 * ncw;
        const bool in_cg = tc >= cg0;
        const int gt = tc - cg0;  // thread index in the colour group
        auto bar_colour = [&]() {
            if (overlap) asm volatile("bar.sync 3, %0;" ::"r"(ng) : "memory");
            else bar_chain();
        };
        bar_chain();
        if (tc == 0) qb_arrive(a);
        if (bl == 0 && tc == 0) a.rec_time[0] = globaltimer_ns();
        double smax = 0.0;  // max |delta| of this thread's own pairs over the sweep
        int snnz = 0;
        long long t_wait = 0, t_load = 0, t_work = 0, t_c0 = 0, t_c3 = 0;
        long long t_q0 = 0, t_q1 = 0, t_q2 = 0;  // colour sub-steps of the thread of the first pair
        // Cells of block B, part A -- everything that does not depend on the deltas of block
        // B-1: layout, stage values (watermark C'(B) = start of block B-3, minus one), in-block
        // T entries and pair slots, and the deltas of blocks B-3, B-2 (phases C'(B)+1 .. g0(B-1)-1).
        // Part B (after the barrier of block B) folds in the deltas of block B-1, in phase
        // order.  Blocks alternate between two cell buffers and two layouts.  Threads
        // [0, gs) take part, synchronised by the named barrier `bar_id`.
        auto cells_a = [&](int B, int gs, int bar_id) {
            const Blk kB = block_at(B, m, D, NB, a.nb_magic, a.nb_shift);
            const bool hdB = (kB.ph0 + kB.len - 1 == m);
            const int nbcB = kB.len - (hdB ? 1 : 0);
            const int CpB = stage_mark(B, m, D, NB, a.nb_magic, a.nb_shift);
            const int hiA = (B >= 1) ? block_at(B - 1, m, D, NB, a.nb_magic, a.nb_shift).g0 : 0;
            const int na = hiA - (CpB + 1);
            Layout& L = s_ly[B & 1];
            const int cb = (a.nbuf == 2) ? (B & 1) * a.cellcap : 0;
            // layout: colour d = 0..nbc-1 covers pairs [lo_d, hi_d), two cells per pair;
            // then the diagonal cells (rows of the own pairs at colour m-1)
            if (tc == 0) {
                int nc = 0;
                for (int d = 0; d < kDMax; ++d) {
                    const int h = nbcB - 1 - d;
                    L.lo[d] = (d < nbcB) ? max(0, q_lo - h) : 0;
                    const int hi = (d < nbcB) ? min(half, q_hi + h) : 0;
                    L.cb[d] = nc;
                    nc += (d < nbcB) ? 2 * (hi - L.lo[d]) : 0;
                }
                L.cb[kDMax] = nc;
                L.ncell = nc;
                // ring slots of the block's phases: one modulo per ring, then wraps (d <= D < ring sizes)
                const int gs0 = kB.g0 % a.sr, gd0 = kB.g0 % a.rd, gl0 = kB.g0 % a.rl;
                for (int d = 0; d <= kDMax; ++d) L.slot[d] = (gs0 + d >= a.sr) ? gs0 + d - a.sr : gs0 + d;
                for (int d = 0; d < kDMax; ++d) {
                    L.rdc[d] = (gd0 + d >= a.rd) ? gd0 + d - a.rd : gd0 + d;
                    L.lsl[d] = (gl0 + d >= a.rl) ? gl0 + d - a.rl : gl0 + d;
                }
            } else if (tc == 1) {  // the delta-walk starts, in parallel with thread 0
                L.rd0 = (CpB + 1) % a.rd;
                L.ph0w = (CpB + 1) % (m + 1);
            } else if (tc == 2) {
                L.rdb = hiA % a.rd;
                L.phb = hiA % (m + 1);
            }
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(gs) : "memory");
            const int ncellB = L.ncell;
            const int ntotB = ncellB + (hdB ? 2 * (q_hi - q_lo) : 0);
            for (int ci = tc; ci < ntotB; ci += gs) {
                int d, x, c;
                if (ci < ncellB) {
                    d = 0;
                    while (d + 1 < nbcB && ci >= L.cb[d + 1]) ++d;
                    const int rel = ci - L.cb[d];
                    const int q = L.lo[d] + (rel >> 1);
                    int r, s2;
                    round_pair(q, m, m - 1 - (kB.ph0 + d), r, s2);
                    if (s2 >= p) {
                        sm.cX()[cb + ci] = -1;
                        continue;
                    }
                    x = (rel & 1) ? s2 : r;
                    c = (rel & 1) ? r : s2;
                } else {
                    d = nbcB;
                    const int rel = ci - ncellB;
                    const int q = q_lo + (rel >> 1);
                    int r, s2;
                    round_pair(q, m, 0, r, s2);  // colour m-1
                    x = (rel & 1) ? s2 : r;
                    if (x >= p) {
                        sm.cX()[cb + ci] = -1;
                        continue;
                    }
                    c = x;
                }
                // column c of T: row-major storage (slabT == w) is plain column indexing
                const double* Tc = (a.slabT == w) ? a.Tfull + c
                                                  : a.Tfull + (long long)(c / w) * a.slabT + (c - (c / w) * w);
                const size_t so = (size_t)L.slot[d] * p + c;
                double val = __ldcg(stWL + so);
                const double om = __ldcg(stOL + so);
                // in-block phases ph0 .. ph0+d-1: T entries staged by the slab owner; the row's
                // pair index (into sd) stepped without division
                double tin[kDMax - 1];
#pragma unroll
                for (int i = 0; i < kDMax - 1; ++i)
                    tin[i] = ldcg_if(stTL + ((size_t)L.slot[d] * (kDMax - 1) + i) * p + c, i < d);
                {
                    int pos = x - 1 + kB.ph0;  // in [0, 2m): one conditional subtraction for the mod
                    pos = (x == 0) ? 0 : 1 + (pos >= m ? pos - m : pos);
                    for (int i = 0; i < d; ++i) {
                        const int qi = (pos == 0 || pos == m) ? 0 : min(pos, m - pos);
                        sm.cQ()[(size_t)(cb + ci) * dm1 + i] = (short)(qi - L.lo[i]);
                        if (x != 0) pos = (pos == m) ? 1 : pos + 1;
                    }
                }
                // deltas of blocks B-3 and B-2: ring loads back to back; T entries (HBM) only for
                // the phases that moved row x, again back to back; then the FMAs in phase order
                double dj[2 * kDMax];
                int slot = L.rd0;
#pragma unroll
                for (int u = 0; u < 2 * kDMax; ++u) {
                    dj[u] = ldcg_if(dringL + (size_t)slot * p + x, u < na);
                    slot = (slot + 1 == a.rd) ? 0 : slot + 1;
                }
                unsigned mask = 0u;
#pragma unroll
                for (int u = 0; u < 2 * kDMax; ++u)
                    if (dj[u] != 0.0) mask |= 1u << u;
                if (mask) {
                    double tj[2 * kDMax];
                    PartnerWalk pw(x, L.ph0w, m);
#pragma unroll
                    for (int u = 0; u < 2 * kDMax; ++u) {
                        tj[u] = ldcg_if(Tc + (long long)pw.y() * a.ldT, (mask >> u) & 1u);
                        pw.next();
                    }
#pragma unroll
                    for (int u = 0; u < 2 * kDMax; ++u)
                        if (mask & (1u << u)) val = fma(dj[u], tj[u], val);
                }
                sm.cX()[cb + ci] = x;
                sm.cC()[cb + ci] = c;
                sm.cW()[cb + ci] = val;
                sm.cO()[cb + ci] = om;
#pragma unroll
                for (int i = 0; i < kDMax - 1; ++i)
                    if (i < dm1) sm.cT()[(size_t)(cb + ci) * dm1 + i] = tin[i];
            }
        };
        int blk = 0;
        while (true) {
            const long long t0 = PCLK();
            const Blk k = block_at(blk, m, D, NB, a.nb_magic, a.nb_shift);
            if (tc == 0) {
                wait_counter(barL, a.bar_base + (unsigned long long)(blk + 1) * (unsigned long long)nblk, blk, a.hang,
                             a.sys_scope);
                st_vol(&s_epoch, k.g0);  // deltas and lists of every phase < g0 are visible
                st_vol(&s_blk, blk);
            }
            bar_chain();
            const long long t1 = PCLK();
            t_wait += t1 - t0;
            // ---- the previous block closed a sweep: convergence decision (identical in every CTA)
            if (k.ph0 == 0 && blk > 0) {
                const int it = k.sweep - 1;
                const double dmax_all =
                    __longlong_as_double((long long)__ldcg(dmaxL + (a.it_base + it) % WFORM_DMAX_RING));
                // a yield request (CTA 0 sampled the host flag before closing the sweep) stops a fit
                // that would go on; the state is then exactly the one after sweep it (resumable)
                const bool yld = __ldcg(dmaxL + WFORM_DMAX_RING + (a.it_base + it) % WFORM_DMAX_RING) != 0ull;
                const bool stop = (dmax_all < a.delta_tol) || (it + 1 >= a.max_iter) || yld;
                if (bl == 0 && tc == 0) {
                    a.rec_delta[it] = dmax_all;
                    a.rec_time[it + 1] = globaltimer_ns();
                }
                if (b == 0 && tc == 0)  // recycle the accumulators of sweep it+2 (last read at sweep it-2)
                    QB_COPIES(r) {
                        a.x.dmax[r][(a.it_base + it + 2) % WFORM_DMAX_RING] = 0ull;
                        a.x.dmax[r][WFORM_DMAX_RING + (a.it_base + it + 2) % WFORM_DMAX_RING] = 0ull;
                    }
                if (stop) {
                    if (tc == 0) {
                        s_iters = it + 1;
                        s_conv = (dmax_all < a.delta_tol) ? 1 : ((it + 1 < a.max_iter && yld) ? 2 : 0);
                        __threadfence_block();
                        st_vol(&s_stop, k.g0 - 1);
                    }
                    break;
                }
            }
            const bool has_diag = (k.ph0 + k.len - 1 == m);
            const int nbc = k.len - (has_diag ? 1 : 0);  // colour phases of the block
            const Layout& L = s_ly[blk & 1];
            const int cb = (a.nbuf == 2) ? (blk & 1) * a.cellcap : 0;
            if (blk == 0) {
                cells_a(0, kChain, 1);
                bar_chain();
            }
            // ---- cells, part B (on the critical path): deltas of the previous block
            {
                const int hiA = (blk >= 1) ? block_at(blk - 1, m, D, NB, a.nb_magic, a.nb_shift).g0 : 0;
                const int nbv = k.g0 - hiA;
                const int ntotB = L.ncell + (has_diag ? 2 * (q_hi - q_lo) : 0);
                // two cells per step: both cells' ring loads, then both cells' T loads, back to back
                for (int c0i = tc; c0i < ntotB; c0i += 2 * kChain) {
                    double dj[2][kDMax];
                    int xs[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int ci = c0i + h * kChain;
                        xs[h] = (ci < ntotB) ? sm.cX()[cb + ci] : -1;
                        int slot = L.rdb;
#pragma unroll
                        for (int u = 0; u < kDMax; ++u) {
                            dj[h][u] = ldcg_if(dringL + (size_t)slot * p + max(xs[h], 0), xs[h] >= 0 && u < nbv);
                            slot = (slot + 1 == a.rd) ? 0 : slot + 1;
                        }
                    }
                    unsigned mask[2] = {0u, 0u};
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int u = 0; u < kDMax; ++u)
                            if (dj[h][u] != 0.0) mask[h] |= 1u << u;
                    if (mask[0] | mask[1]) {
                        double tj[2][kDMax];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int ci = c0i + h * kChain;
                            const int c = mask[h] ? sm.cC()[cb + ci] : 0;
                            const double* Tc = (a.slabT == w)
                                                   ? a.Tfull + c
                                                   : a.Tfull + (long long)(c / w) * a.slabT + (c - (c / w) * w);
                            PartnerWalk pw(max(xs[h], 0), L.phb, m);
#pragma unroll
                            for (int u = 0; u < kDMax; ++u) {
                                tj[h][u] = ldcg_if(Tc + (long long)pw.y() * a.ldT, (mask[h] >> u) & 1u);
                                pw.next();
                            }
                        }
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (!mask[h]) continue;
                            const int ci = c0i + h * kChain;
                            double val = sm.cW()[cb + ci];
#pragma unroll
                            for (int u = 0; u < kDMax; ++u)
                                if (mask[h] & (1u << u)) val = fma(dj[h][u], tj[h][u], val);
                            sm.cW()[cb + ci] = val;
                        }
                    }
                }
            }
            bar_chain();
            const int ncell = L.ncell;
            const int ndiag = has_diag ? 2 * (q_hi - q_lo) : 0;
            const long long t2 = PCLK();
            t_load += t2 - t1;

            if (in_cg) {
                // ---- the block's colours, in order, in shared memory; only the deltas (sd) and
                // the new values of the own pairs (snv) are written per colour, the ring and the
                // lists after the last colour
                for (int d = 0; d < nbc; ++d) {
                    const int ph = k.ph0 + d;
                    const int h = nbc - 1 - d;
                    const int hi = min(half, q_hi + h);
                    const int lod = L.lo[d], cbd = cb + L.cb[d];
                    const int c1 = m - 1 - ph;
                    double* sdd = sm.sd() + (size_t)d * a.rmax;
                    const int sid = ng - 1 - gt;
                    for (int base = lod; base < hi; base += ng) {
                        const int q = base + sid;
                        if (q >= hi) continue;
                        long long tp0 = 0, tp1 = 0, tp2 = 0;
                        if (prof && sid == 0) tp0 = PCLK();
                        int r, s;
                        round_pair(q, m, c1, r, s);
                        double dl = 0.0, nv = 0.0;
                        if (s < p) {
                            const int ci = cbd + 2 * (q - lod);
                            // corrections of the block's earlier colours, three rounds of shared
                            // loads (pair slots, deltas, T entries) for both cells, then the FMAs
                            // in colour order
                            short qi[2][kDMax - 1];
                            double di[2][kDMax - 1], ti[2][kDMax - 1], v2[2];
#pragma unroll
                            for (int side = 0; side < 2; ++side) {
                                v2[side] = sm.cW()[ci + side];
#pragma unroll
                                for (int i = 0; i < kDMax - 1; ++i)
                                    qi[side][i] = (i < d) ? sm.cQ()[(size_t)(ci + side) * dm1 + i] : (short)0;
                            }
#pragma unroll
                            for (int side = 0; side < 2; ++side)
#pragma unroll
                                for (int i = 0; i < kDMax - 1; ++i) {
                                    di[side][i] = (i < d) ? sm.sd()[(size_t)i * a.rmax + qi[side][i]] : 0.0;
                                    ti[side][i] = (i < d) ? sm.cT()[(size_t)(ci + side) * dm1 + i] : 0.0;
                                }
#pragma unroll
                            for (int side = 0; side < 2; ++side)
#pragma unroll
                                for (int i = 0; i < kDMax - 1; ++i)
                                    if (i < d && di[side][i] != 0.0) v2[side] = fma(di[side][i], ti[side][i], v2[side]);
                            // side 0: cell (r, s) = W[r,s]; side 1: cell (s, r) = W[s,r]
                            const double om = sm.cO()[ci];
                            if (prof && sid == 0) tp1 = clock_after(v2[0] + v2[1]);
                            dl = pair_delta(make_double2(v2[1], om), make_double2(v2[0], om), TD(r), TD(s), a.shrink,
                                            nv);
                            if (prof && sid == 0) tp2 = clock_after(dl);
                        }
                        sdd[q - lod] = dl;
                        if (q >= q_lo && q < q_hi) sm.snv()[d * a.share + (q - q_lo)] = nv;
                        if (prof && sid == 0 && tp2 != 0) {
                            const long long tp3 = PCLK();
                            t_q0 += tp1 - tp0;
                            t_q1 += tp2 - tp1;
                            t_q2 += tp3 - tp2;
                        }
                    }
                    bar_colour();
                }
                // ---- publish the own pairs of all colours: delta ring, non-zero delta lists
                {
                    const int nown = q_hi - q_lo;
                    const int nwn = max(nown, 1);
                    // item (colour d, own pair q) stepped without division
                    const int pdq = ng / nwn, pdr = ng - pdq * nwn;
                    int pd = gt / nwn, pr = gt - (gt / nwn) * nwn;
                    for (int base = 0; base < nbc * nown; base += ng) {
                        const int idx = base + gt;
                        const bool live = idx < nbc * nown;
                        int d = 0, q = 0, r = 0, s = 0;
                        double dl = 0.0, nv = 0.0;
                        const int d_it = pd, r_it = pr;
                        pd += pdq;
                        pr += pdr;
                        if (pr >= nwn) {
                            pr -= nwn;
                            ++pd;
                        }
                        if (live) {
                            d = d_it;
                            q = q_lo + r_it;
                            round_pair(q, m, m - 1 - (k.ph0 + d), r, s);
                            dl = sm.sd()[(size_t)d * a.rmax + (q - L.lo[d])];
                            nv = sm.snv()[d * a.share + (q - q_lo)];
                            const size_t dgo = (size_t)L.rdc[d] * p;
                            QB_COPIES(cp) {
                                a.x.dring[cp][dgo + r] = dl;  // 0 when the partner is the phantom (odd p)
                                if (s < p) a.x.dring[cp][dgo + s] = dl;
                            }
                            if (dl != 0.0) {
                                smax = fmax(smax, abs_delta(dl));
                                ++snnz;
                            }
                        }
                        const bool nz = live && dl != 0.0;
                        // one warp-aggregated slot reservation per colour present in the warp
                        unsigned pending = __ballot_sync(0xffffffffu, nz);
                        int at = 0;
                        while (pending) {
                            const int leader = __ffs(pending) - 1;
                            const int dd = __shfl_sync(0xffffffffu, d, leader);
                            const unsigned mm = __ballot_sync(0xffffffffu, nz && d == dd);
                            int basepos = 0;
                            if (lane == leader) basepos = atomicAdd(&s_cnt[dd], __popc(mm));
                            basepos = __shfl_sync(0xffffffffu, basepos, leader);
                            if (nz && d == dd) at = basepos + __popc(mm & ((1u << lane) - 1u));
                            pending &= ~mm;
                        }
                        if (nz) {
                            const size_t seg_off = ((size_t)L.lsl[d] * nblk + b) * a.share;
                            QB_COPIES(cp) {
                                a.x.list_rs[cp][seg_off + at] = make_int2(r, s);
                                a.x.list_dn[cp][seg_off + at] = make_double2(dl, nv);
                            }
                        }
                    }
                    bar_colour();
                    if (gt == 0) {  // the thread that arrives: its own stores are ordered by the release
                        for (int d = 0; d < nbc; ++d) {
                            const int cnt_d = s_cnt[d];
                            QB_COPIES(cp) a.x.list_cnt[cp][(size_t)L.lsl[d] * nblk + b] = cnt_d;
                            s_cnt[d] = 0;
                        }
                    }
                }

                // ---- diagonal phase (closes the sweep): rows of the own pairs at colour m-1
                if (has_diag) {
                    const int Qd = k.g0 + nbc;
                    const size_t dgo = (size_t)(Qd % a.rd) * p;
                    double dm = 0.0;
                    for (int e = gt; e < ndiag; e += ng) {
                        const int cc = cb + ncell + e;
                        const int x = sm.cX()[cc];
                        if (x < 0) continue;
                        double val = sm.cW()[cc];
                        for (int i = 0; i < nbc; ++i) {
                            const double di = sm.sd()[(size_t)i * a.rmax + sm.cQ()[(size_t)cc * dm1 + i]];
                            if (di != 0.0) val = fma(di, sm.cT()[(size_t)cc * dm1 + i], val);
                        }
                        const double om = sm.cO()[cc];
                        const double nv = diag_from_dot(val, om, TD(x), a.n);
                        const double dl = __dsub_rn(nv, om);
                        QB_COPIES(cp) {
                            a.x.dring[cp][dgo + x] = dl;
                            a.x.diagv[cp][x] = make_double2(dl, nv);
                        }
                        dm = fmax(dm, abs_delta(dl));
                    }
                    // this sweep's statistics: off-diagonal (own pairs) and diagonal maxima, non-zero count
                    const double mw = warp_max(fmax(dm, smax));
                    const double nw = warp_sum((double)snnz);
                    if (lane == 0) {
                        s_red[0][warp] = mw;
                        s_red[1][warp] = nw;
                    }
                    smax = 0.0;
                    snnz = 0;
                    bar_colour();
                    if (gt == 0) {
                        double mb = 0.0, nbk = 0.0;
                        for (int j = cg0 / 32; j < kChainWarps; ++j) {
                            mb = fmax(mb, s_red[0][j]);
                            nbk += s_red[1][j];
                        }
                        QB_COPIES(cp)
                            atomicMax(a.x.dmax[cp] + (a.it_base + k.sweep) % WFORM_DMAX_RING,
                                      (unsigned long long)__double_as_longlong(mb));
                        if (b == 0 && a.yield != nullptr && *a.yield != 0)
                            QB_COPIES(cp) a.x.dmax[cp][WFORM_DMAX_RING + (a.it_base + k.sweep) % WFORM_DMAX_RING] = 1ull;
                        atomicAdd(reinterpret_cast<unsigned long long*>(a.rec_nnz + k.sweep), (unsigned long long)nbk);
                    }
                }
                if (gt == 0) t_work += PCLK() - t2;
                // ---- the block after next must be staged (by this CTA's apply warps) before
                // arriving: part A of the next block's cells reads it before that block's barrier
                if (gt == 0) {
                    const long long tw0 = PCLK();
                    const unsigned long long g0t = globaltimer_ns();
                    while (ld_acquire_cta(&s_staged) < blk + 2) {
                        if (QB_POLL_NS) __nanosleep(QB_POLL_NS);
                        if (globaltimer_ns() - g0t > kHangNs) hang_report(a.hang, 1, blk, blk + 2, ld_vol(&s_staged), 0, 0);
                    }
                    t_c3 += PCLK() - tw0;
                    qb_arrive(a);
                }
            }
            // ---- part A of the next block's cells: the prefetch group, concurrently with the
            // colours (or every chain warp, after the arrive)
            if (overlap ? !in_cg : true) {
                const long long ta0 = PCLK();
                cells_a(blk + 1, overlap ? cg0 : kChain, overlap ? 4 : 1);
                t_c0 += PCLK() - ta0;
            }
            bar_chain();
            ++blk;
        }
        if (prof && tc == 0) {
            prof[0] = (unsigned long long)t_wait;
            prof[1] = (unsigned long long)t_load;
            prof[3] = (unsigned long long)blk;
            prof[7] = (unsigned long long)t_c0;
        }
        if (prof && tc == cg0) {
            prof[2] = (unsigned long long)t_work;
            prof[9] = (unsigned long long)t_c3;
        }
        if (prof && tc == kChain - 1) {
            prof[12] = (unsigned long long)t_q0;
            prof[13] = (unsigned long long)t_q1;
            prof[14] = (unsigned long long)t_q2;
        }
    } else {
#if QB_NS_REGS_APPLY
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(QB_NS_REGS_APPLY));
#endif
        // ================================================================ apply warps
        const int ta = tid - kChain;
        int C = -1;    // every phase <= C is in the own slab
        int cph = m;   // phase-in-sweep of C
        int cit = -1;  // sweep of C
        int staged = 1;  // highest block staged
        long long t_busy = 0, t_idle = 0, nbatch = 0, t_diag = 0, t_stage = 0, t_heads = 0, t_rows = 0;
        unsigned long long idle_since = 0;  // watchdog (thread ta == 0)
        int last_total = 0;                 // entries of the previous colour batch
        while (true) {
            const long long t0 = PCLK();
            bar_apply();
            if (ta == 0) {
                s_aE = ld_vol(&s_epoch);
                s_aBlk = ld_vol(&s_blk);
                s_aStop = ld_vol(&s_stop);
                s_nent = 0;
                s_multi = 0;
                s_conflict = 0;
                __threadfence_block();
            }
            bar_apply();
            const long long th0 = PCLK();
            const int E = s_aE;
            const int cblk = s_aBlk;
            const int stopg = s_aStop;
            const int avail = (stopg >= 0) ? stopg : E - 1;
            const int k0 = C + 1;
            const int ph0 = (cph == m) ? 0 : cph + 1;
            const int it0 = (cph == m) ? cit + 1 : cit;
            const bool have = C < avail;
            const bool diag = have && ph0 == m;
            const int k1 = (have && !diag) ? min(min(avail, k0 + kBatch - 1), k0 + (m - 1 - ph0)) : C;
            const int nb = k1 - C;
            const int nsh = nblk;
            const int nseg = nb * nsh;
            // next block to stage: the chain at block cblk needs block cblk+2 before arriving;
            // stage up to cblk+3.  Its watermark C' must be <= E-1 (deltas known) and the
            // window (C, C'] must still be in the delta ring.
            const int sb = staged + 1;
            const int Cp = stage_mark(sb, m, D, NB, a.nb_magic, a.nb_shift);
            const bool can_stage = stopg < 0 && cblk >= 0 && sb <= cblk + 3 && Cp <= E - 1 && C >= Cp - a.stage_window;
            // and the block after it in the same pass when it is eligible too and the batches are
            // small (the apply then gets a block ahead of the chain's needs and its latency-bound
            // batches grow to two blocks; dense batches are bandwidth-bound and gain nothing)
            const int Cp2 = stage_mark(sb + 1, m, D, NB, a.nb_magic, a.nb_shift);
            const bool can2 = can_stage && last_total <= 256 && sb + 1 <= cblk + 3 && Cp2 <= E - 1 &&
                              C >= Cp2 - a.stage_window;
            if (!have && !can_stage) {
                t_idle += PCLK() - t0;
                // the chain stopped after this slab already reached the last phase: done
                if (stopg >= 0 && C >= stopg) break;
                if (ta == 0) {
                    if (idle_since == 0) idle_since = globaltimer_ns();
                    else if (globaltimer_ns() - idle_since > kHangNs) hang_report(a.hang, 2, cblk, C, E, staged, stopg);
                }
                if (QB_IDLE_NS) __nanosleep(QB_IDLE_NS);
                continue;
            }
            idle_since = 0;

            // ---- segment heads (count + first entry) of the batch's colours: copied
            // asynchronously into shared memory while this thread stages (below); every
            // thread then reads back only the heads it copied
            // segment (batch phase jb, CTA) stepped without division; ring slot of phase k0 + jb
            const int k0rl = k0 % a.rl;
            const int hsq = kApply / nsh, hsr = kApply - hsq * nsh;
            int hjb = ta / nsh, hcta = ta - (ta / nsh) * nsh;
            for (int idx = ta; idx < nseg; idx += kApply) {
                const int jb = hjb;
                const int slot = (k0rl + jb >= a.rl) ? k0rl + jb - a.rl : k0rl + jb;
                const int seg = slot * nblk + hcta;
                hjb += hsq;
                hcta += hsr;
                if (hcta >= nsh) {
                    hcta -= nsh;
                    ++hjb;
                }
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (unsigned)__cvta_generic_to_shared(sm.s_off() + idx)),
                             "l"(lcntL + seg)
                             : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                 (unsigned)__cvta_generic_to_shared(sm.hd_rs() + idx)),
                             "l"(lrsL + (size_t)seg * a.share)
                             : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 (unsigned)__cvta_generic_to_shared(sm.hd_dn() + idx)),
                             "l"(ldnL + (size_t)seg * a.share)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            // ---- stage block sb: cells brought forward from this slab's watermark C to C'
            if (can_stage) {
                const long long ts = PCLK();
                const Blk kb0 = block_at(sb, m, D, NB, a.nb_magic, a.nb_shift);
                const Blk kb1 = block_at(sb + 1, m, D, NB, a.nb_magic, a.nb_shift);
                const int n0 = kb0.len * wl;
                const int nst = n0 + (can2 ? kb1.len * wl : 0);
                // cell (phase i of the block, slab column j) stepped without division; the ring slots
                // of the delta walk and the block's stage slots hoisted out of the loop
                const int rslot0 = (C + 1) % a.rd, phw0 = (C + 1) % (m + 1);
                const int sl0 = kb0.g0 % a.sr, sl1 = kb1.g0 % a.sr;  // stage slots of the blocks' first phases
                const int wld = max(wl, 1);  // a padding slab (no columns) runs no iterations
                const int sq = kApply / wld, sr = kApply - sq * wld;
                int ci = ta / wld, cj = ta - (ta / wld) * wld;
                bool second = false;
                for (int idx2 = ta; idx2 < nst; idx2 += kApply) {
                    if (!second && idx2 >= n0) {
                        second = true;
                        ci = (idx2 - n0) / wld;
                        cj = (idx2 - n0) - ci * wld;
                    }
                    const int i = ci, j = cj;
                    ci += sq;
                    cj += sr;
                    if (cj >= wld) {
                        cj -= wld;
                        ++ci;
                    }
                    const Blk kb = second ? kb1 : kb0;
                    const int Cpx = second ? Cp2 : Cp;
                    int qs = (second ? sl1 : sl0) + i;  // stage slot of phase kb.g0 + i (i < D < sr)
                    qs -= (qs >= a.sr) ? a.sr : 0;
                    const int c = c0 + j;
                    const int x = pub_row(kb.ph0 + i, c, m, p);
                    if (x < 0) continue;
                    double val = __ldcg(Wb + (long long)x * ld + j);
                    const double om = __ldcg(Ob + (long long)x * ld + j);
                    // deltas of phases C+1 .. Cpx, eight at a time: ring loads back to back, then the
                    // T entries of the phases that moved row x (predicated, back to back), then the FMAs
                    int rslot = rslot0;
                    PartnerWalk pw(x, phw0, m);
                    for (int j0 = C + 1; j0 <= Cpx; j0 += 8) {
                        double dj[8], tj[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            dj[u] = ldcg_if(dringL + (size_t)rslot * p + x, j0 + u <= Cpx);
                            rslot = (rslot + 1 == a.rd) ? 0 : rslot + 1;
                        }
                        unsigned mk = 0u;
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (dj[u] != 0.0) mk |= 1u << u;
                        if (mk) {
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                tj[u] = ldcg_if(Tb + (long long)pw.y() * ld + j, (mk >> u) & 1u);
                                pw.next();
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (mk & (1u << u)) val = fma(dj[u], tj[u], val);
                        } else {
#pragma unroll
                            for (int u = 0; u < 8; ++u) pw.next();
                        }
                    }
                    const size_t so = (size_t)qs * p + c;
                    QB_COPIES(cp) {
                        a.x.stW[cp][so] = val;
                        a.x.stO[cp][so] = om;
                    }
                    // T entries of the block's earlier phases (kb.ph0 .. ph-1), for the chain's in-block
                    // FMAs: all loads first (predicated, back to back), then the stores
                    {
                        double tv[kDMax - 1];
                        PartnerWalk pt(x, kb.ph0, m);
#pragma unroll
                        for (int ii = 0; ii < kDMax - 1; ++ii) {
                            const int y = pt.y();
                            tv[ii] = ldcg_if(Tb + (long long)min(y, p - 1) * ld + j, ii < i && y < p);
                            pt.next();
                        }
#pragma unroll
                        for (int ii = 0; ii < kDMax - 1; ++ii)
                            if (ii < i) QB_COPIES(cp) a.x.stT[cp][((size_t)qs * (kDMax - 1) + ii) * p + c] = tv[ii];
                    }
                }
                t_stage += PCLK() - ts;
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            hjb = ta / nsh;
            hcta = ta - hjb * nsh;
            for (int idx = ta; idx < nseg; idx += kApply) {
                const int jb = hjb;
                hjb += hsq;
                hcta += hsr;
                if (hcta >= nsh) {
                    hcta -= nsh;
                    ++hjb;
                }
                const int cnt = sm.s_off()[idx];
                if (cnt > 1) s_multi = 1;
                if (cnt == 1) {
                    const int2 rs = sm.hd_rs()[idx];
                    const double2 dn = sm.hd_dn()[idx];
                    const int pos = atomicAdd(&s_nent, 1);
                    if (pos < kPairCap) {
                        sm.L_rs()[pos] = rs;
                        sm.L_d()[pos] = dn.x;
                        sm.L_ph()[pos] = jb;
                    } else {
                        s_multi = 1;
                    }
                    if ((unsigned)(rs.y - c0) < (unsigned)wl) Ob[(long long)rs.x * ld + (rs.y - c0)] = dn.y;
                    if ((unsigned)(rs.x - c0) < (unsigned)wl) Ob[(long long)rs.y * ld + (rs.x - c0)] = dn.y;
                }
            }
            bar_apply();
            const long long th1 = PCLK();
            if (can_stage) {
                staged = can2 ? sb + 1 : sb;
                if (ta == 0) {
                    __threadfence_block();
                    st_vol(&s_staged, staged);
                }
            }

            if (diag) {
                // ---- dense diagonal step over the own slab (+ objective records)
                const double2* dd = diagvL;
                double q_acc = 0.0, pen_acc = 0.0, log_acc = 0.0;
                for (int i0 = 0; i0 < p; i0 += kPairCap) {
                    const int iend = min(i0 + kPairCap, p);
                    for (int i = i0 + ta; i < iend; i += kApply) {
                        const double2 v = ldcg2(dd + i);
                        sm.L_d()[i - i0] = v.x;
                        sm.L_new()[i - i0] = v.y;
                    }
                    bar_apply();
                    const int items = (iend - i0) * w2;
                    // item (row ii of the chunk, column pair j2) of each unrolled slot, stepped
                    // without division
                    int cii[kUnroll], cjj[kUnroll];
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        cii[u] = (u * kApply + ta) / w2;
                        cjj[u] = (u * kApply + ta) - cii[u] * w2;
                    }
                    const int dsq = (kApply * kUnroll) / w2, dsr = kApply * kUnroll - dsq * w2;
                    for (int base = 0; base < items; base += kApply * kUnroll) {
                        double2 wv[kUnroll], tv[kUnroll], ov[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int idx = base + u * kApply + ta;
                            if (idx < items) {
                                const int ii = cii[u];
                                const int j2 = cjj[u];
                                const long long off = (long long)(i0 + ii) * ld + 2 * j2;
                                wv[u] = __ldcg(reinterpret_cast<const double2*>(Wb + off));
                                if (sm.L_d()[ii] != 0.0) tv[u] = __ldcg(reinterpret_cast<const double2*>(Tb + off));
                                if (a.want_trace) ov[u] = *reinterpret_cast<const double2*>(Ob + off);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int idx = base + u * kApply + ta;
                            if (idx < items) {
                                const int ii = cii[u];
                                const int j2 = cjj[u];
                                const int i = i0 + ii;
                                const long long off = (long long)i * ld + 2 * j2;
                                const double d = sm.L_d()[ii];
                                if (d != 0.0) {
                                    wv[u].x = fma(d, tv[u].x, wv[u].x);
                                    wv[u].y = fma(d, tv[u].y, wv[u].y);
                                    *reinterpret_cast<double2*>(Wb + off) = wv[u];
                                }
                                const int cj = c0 + 2 * j2;
                                const bool dg0 = (cj == i), dg1 = (cj + 1 == i);
                                if (a.want_trace) {
                                    if (dg0 | dg1) {
                                        if (dg0) ov[u].x = sm.L_new()[ii];
                                        if (dg1) ov[u].y = sm.L_new()[ii];
                                        *reinterpret_cast<double2*>(Ob + off) = ov[u];
                                        log_acc += log(sm.L_new()[ii]);
                                    }
                                    q_acc = fma(wv[u].x, ov[u].x, q_acc);
                                    q_acc = fma(wv[u].y, ov[u].y, q_acc);
                                    if (i < cj) pen_acc += fabs(ov[u].x);
                                    if (i < cj + 1) pen_acc += fabs(ov[u].y);
                                } else if (dg0 | dg1) {
                                    Ob[off + (dg0 ? 0 : 1)] = sm.L_new()[ii];
                                }
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            cii[u] += dsq;
                            cjj[u] += dsr;
                            if (cjj[u] >= w2) {
                                cjj[u] -= w2;
                                ++cii[u];
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
                t_heads += th1 - th0;
                const long long tr0 = PCLK();
                int total = 0;
                if (!s_multi) {
                    // every segment had at most one entry: they are already in shared memory
                    const int nent = s_nent;
                    if (nb > 1) {
                        for (int e = ta; e < nent; e += kApply) {
                            const int2 rs = sm.L_rs()[e];
                            const unsigned br = 1u << (rs.x & 31), bs = 1u << (rs.y & 31);
                            const unsigned o1 = atomicOr(sm.bm() + (rs.x >> 5), br);
                            const unsigned o2 = atomicOr(sm.bm() + (rs.y >> 5), bs);
                            if ((o1 & br) | (o2 & bs)) s_conflict = 1;
                        }
                        bar_apply();
                    }
                    if (!s_conflict) {
                        ROWS(sm.L_rs(), sm.L_d(), sm.L_ph(), -1, 0, nent, w2, Wb, Tb, sm.ring(), ta);
                    } else if (nent <= kChainN) {
                        apply_chains(sm.L_rs(), sm.L_d(), sm.L_ph(), nent, w2, a.w2_magic, a.w2_shift, ld2, Wb, Tb, s_next, s_first,
                                     ta);
                    } else {
                        for (int jb = 0; jb < nb; ++jb) {  // rows repeat across phases: phase by phase
                            ROWS(sm.L_rs(), sm.L_d(), sm.L_ph(), jb, 0, nent, w2, Wb, Tb, sm.ring(), ta);
                            bar_apply();
                        }
                    }
                    bar_apply();
                    if (nb > 1) {
                        for (int e = ta; e < nent; e += kApply) {
                            const int2 rs = sm.L_rs()[e];
                            atomicAnd(sm.bm() + (rs.x >> 5), ~(1u << (rs.x & 31)));
                            atomicAnd(sm.bm() + (rs.y >> 5), ~(1u << (rs.y & 31)));
                        }
                    }
                    total = nent;
                } else {
                    // general path: exclusive scan of the segment counts, entries in phase order
                    total = apply_scan(sm.s_off(), nseg, ta, s_wsum);
                    for (int e0 = 0; e0 < total; e0 += kPairCap) {
                        const int e1 = min(total, e0 + kPairCap);
                        for (int e = e0 + ta; e < e1; e += kApply) {
                            int lo = 0, hi = nseg;  // segment: s_off[lo] <= e < s_off[lo+1]
                            while (hi - lo > 1) {
                                const int mid = (lo + hi) >> 1;
                                if (sm.s_off()[mid] <= e) lo = mid;
                                else hi = mid;
                            }
                            const int jb = div_nb(lo, a.nblk_magic, a.nblk_shift);  // lo / nsh
                            const int rank = e - sm.s_off()[lo];
                            const int slot = (k0rl + jb >= a.rl) ? k0rl + jb - a.rl : k0rl + jb;
                            const size_t at = ((size_t)slot * nblk + (lo - jb * nsh)) * a.share + rank;
                            const int2 rs = __ldcg(lrsL + at);
                            const double2 dn = __ldcg(ldnL + at);
                            // segments with one entry had their Omega cells written above
                            if (sm.s_off()[lo + 1] - sm.s_off()[lo] > 1) {
                                if ((unsigned)(rs.y - c0) < (unsigned)wl) Ob[(long long)rs.x * ld + (rs.y - c0)] = dn.y;
                                if ((unsigned)(rs.x - c0) < (unsigned)wl) Ob[(long long)rs.y * ld + (rs.x - c0)] = dn.y;
                            }
                            sm.L_rs()[e - e0] = rs;
                            sm.L_d()[e - e0] = dn.x;
                            sm.L_ph()[e - e0] = jb;
                            if (nb > 1) {
                                const unsigned br = 1u << (rs.x & 31), bs = 1u << (rs.y & 31);
                                const unsigned o1 = atomicOr(sm.bm() + (rs.x >> 5), br);
                                const unsigned o2 = atomicOr(sm.bm() + (rs.y >> 5), bs);
                                if ((o1 & br) | (o2 & bs)) s_conflict = 1;
                            }
                        }
                        bar_apply();
                        const int conflict = s_conflict;
                        if (!conflict) {
                            ROWS(sm.L_rs(), sm.L_d(), sm.L_ph(), -1, 0, e1 - e0, w2, Wb, Tb, sm.ring(), ta);
                        } else if (e1 - e0 <= kChainN) {
                            // few entries: per-row chains, one round trip instead of one pass per phase
                            apply_chains(sm.L_rs(), sm.L_d(), sm.L_ph(), e1 - e0, w2, a.w2_magic, a.w2_shift, ld2, Wb, Tb,
                                         s_next, s_first, ta);
                        } else {
                            for (int jb = 0; jb < nb; ++jb) {
                                const int lo = max(sm.s_off()[jb * nsh], e0) - e0;
                                const int hi = min(sm.s_off()[(jb + 1) * nsh], e1) - e0;
                                if (lo < hi) {  // uniform across the apply warps: no pass, no barrier
                                    ROWS(sm.L_rs(), sm.L_d(), sm.L_ph(), -1, lo, hi, w2, Wb, Tb, sm.ring(), ta);
                                    bar_apply();
                                }
                            }
                        }
                        bar_apply();
                        if (nb > 1) {
                            for (int e = ta; e < e1 - e0; e += kApply) {
                                const int2 rs = sm.L_rs()[e];
                                atomicAnd(sm.bm() + (rs.x >> 5), ~(1u << (rs.x & 31)));
                                atomicAnd(sm.bm() + (rs.y >> 5), ~(1u << (rs.y & 31)));
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
                last_total = total;
                t_rows += PCLK() - tr0;
            }
            t_busy += PCLK() - t0;
            if (stopg >= 0 && C >= stopg) break;
        }
        if (prof && ta == 0) {
            prof[4] = (unsigned long long)t_busy;
            prof[5] = (unsigned long long)t_idle;
            prof[6] = (unsigned long long)nbatch;
            prof[10] = (unsigned long long)t_stage;
            prof[11] = (unsigned long long)t_diag;
            prof[8] = (unsigned long long)t_heads;
            prof[15] = (unsigned long long)t_rows;
        }
    }
#undef TD
    __syncthreads();
    if (bl == 0 && tid == 0) {
        a.status[0] = s_iters;
        a.status[1] = s_conv;
    }
}

#undef PCLK

// Host side of this variant (QB_NS_CHAIN_WARPS chain warps).
size_t smem_bytes(int p, int nblk, int share, int D, int tdiag_smem, int nbuf, int ring_stages) {
    auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
    const size_t cap = (size_t)nbuf * qblock_cellcap(share, D);  // cell buffers
    size_t b = 0;
    b += al(sizeof(int2) * kPairCap) + 2 * al(sizeof(double) * kPairCap) + al(sizeof(int) * kPairCap);
    b += al(sizeof(int) * ((size_t)kBatch * nblk + 1));
    b += al(sizeof(unsigned) * (size_t)((p + 31) / 32));
    b += 2 * al(sizeof(int) * cap) + 2 * al(sizeof(double) * cap) + al(sizeof(double) * cap * (D - 1));
    b += al(sizeof(double) * (size_t)kDMax * qblock_rmax(share, D));
    b += al(sizeof(short) * cap * (D - 1));
    b += al(sizeof(double) * (size_t)kDMax * share);
    b += al(sizeof(int2) * (size_t)kBatch * nblk) + al(sizeof(double2) * (size_t)kBatch * nblk);
    b += al(sizeof(double2) * 2 * (size_t)kApply * ring_stages);
    if (tdiag_smem) b += al(sizeof(double) * (size_t)p);
    return b;
}

// Warps of the colour group for a CTA share (the chain warps the colours need).
int colour_warps_host(int share, int D) { return colour_warps(share, D); }

const void* kernel_fn(bool prof, bool shard) {
    return prof ? (shard ? (const void*)pcd_qblock_kernel<true, true> : (const void*)pcd_qblock_kernel<true, false>)
                : (shard ? (const void*)pcd_qblock_kernel<false, true> : (const void*)pcd_qblock_kernel<false, false>);
}

// Raise the kernel's shared-memory limit only when needed: setting a function attribute while
// another fit runs the kernel on another stream waits for that fit, so solvers reserve their
// launch's bytes when they are created (reserve_smem), not at their first launch.
cudaError_t raise_smem(size_t smem, bool prof, bool shard) {
    static std::mutex mu;
    static size_t set_bytes[4] = {0, 0, 0, 0};
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set_bytes[(prof ? 2 : 0) + (shard ? 1 : 0)];
    if (smem > cur) {
        cudaError_t e = cudaFuncSetAttribute(kernel_fn(prof, shard), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        cur = smem;
    }
    return cudaSuccess;
}

cudaError_t reserve_smem(size_t smem) {
    for (int v = 0; v < 4; ++v) {
        cudaError_t e = raise_smem(smem, v >= 2, v & 1);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch(const QbArgs& args, int nblk, cudaStream_t st) {
    const size_t smem =
        smem_bytes(args.p, args.nblk_tot, args.share, args.D, args.tdiag_smem, args.nbuf, args.ring_stages);
    const bool shard = args.G > 1;
    const void* fn = kernel_fn(args.prof != nullptr, shard);
    {
        cudaError_t e = raise_smem(smem, args.prof != nullptr, shard);
        if (e != cudaSuccess) return e;
    }
    QbArgs copy = args;
    void* kargs[] = {&copy};
    return cudaLaunchCooperativeKernel(fn, dim3(nblk), dim3(kThreads), kargs, smem, st);
}

}  // namespace QB_NS
}  // namespace concord
