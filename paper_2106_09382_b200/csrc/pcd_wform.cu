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
// owns columns [b*w, b*w+w); slab b is a p x w row-major block.  A pair's row
// update only touches a CTA's own columns, so each colour needs ONE grid
// barrier: owners publish (W[partner(c), c], Omega[partner(c), c]) for their
// columns c into a ping-pong buffer, barrier, then every CTA recomputes all
// p/2 closed forms of the colour redundantly (identical arithmetic, so
// identical results in every CTA) and applies the non-zero ones to its slab.
// The max |delta| convergence metric (solver.py:287) is therefore identical in
// every CTA and the stop test needs no extra reduction.  The diagonal phase
// (_ckernels.pyx:96-102) is one dense slab stream that also folds in the
// objective trace (model.py:210-217) as 1/2 <W, Omega>.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "pcd_wform.h"

namespace concord {

constexpr int kThreads = WFORM_THREADS;
constexpr int kCap = WFORM_LIST_CAP;  // list entries (pairs) / diag rows per chunk
constexpr int kUnroll = 2;            // independent row-stream items per thread in flight
constexpr int kMaxBlocks = WFORM_MAX_BLOCKS;

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

__device__ __forceinline__ double diag_delta(double2 v, double tii, double n) {
    return __dsub_rn(diag_from_dot(v.x, v.y, tii, n), v.y);
}

// Row published for column c in phase ph (ph < m: colour ph, ph == m: diagonal), or -1.
__device__ __forceinline__ int pub_row(int ph, int c, int m, int p) {
    const int x = (ph < m) ? circle_partner(c, ph, m) : c;
    return x < p ? x : -1;
}

// Row whose value moves row x in phase ph (its pair partner; x itself on the diagonal).
__device__ __forceinline__ int src_row(int ph, int x, int m) { return ph < m ? circle_partner(x, ph, m) : x; }

// Phase-ph delta of row x (paired with y) recomputed from that phase's publish buffer.
__device__ __forceinline__ double row_delta(int ph, int x, int y, const double2* pb, const double* tdiag, int m,
                                            double shrink, double n, double& nv) {
    if (ph < m) {
        const int r = min(x, y), s = max(x, y);
        return pair_delta(ldcg2(pb + r), ldcg2(pb + s), __ldg(tdiag + r), __ldg(tdiag + s), shrink, nv);
    }
    const double2 v = ldcg2(pb + x);
    nv = diag_from_dot(v.x, v.y, __ldg(tdiag + x), n);
    return __dsub_rn(nv, v.y);
}

__device__ __forceinline__ void bar_arrive(unsigned long long* ctr) {
    // caller has done __syncthreads(); the fence makes the CTA's writes visible first
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1ull);
    }
}

__device__ __forceinline__ void bar_wait(const unsigned long long* ctr, unsigned long long target) {
    if (threadIdx.x == 0) {
        while (ld_acquire_u64(ctr) < target) {
        }
    }
    __syncthreads();
}

// One grid barrier per phase (phase = one colour, or the diagonal step), with
// the work split so that only a few hundred cycles sit between a barrier
// release and the next arrive:
//
//   wait(G)       publishes of phase G (and the delta lists of phase G-1) are visible
//   publish G+1   each column owner publishes (W[x,c], Om[x,c]) of its next cell;
//                 the value was prefetched two phases ago and is brought forward
//                 with the phase G-1 and phase G deltas of row x (recomputed from
//                 the publish buffers: two closed forms and two FMAs, bitwise the
//                 values the bulk row streams produce)
//   share G       the CTA evaluates ITS 1/nblk of the colour's closed forms and
//                 writes the non-zero (r, s, delta, new) to its list segment
//   arrive(G+1)
//   apply G-1     stream the previous phase's non-zero rows into the own slab --
//                 after the arrive, i.e. overlapped with the barrier
//   prefetch      the cell the next publish needs
//
// Publish buffers and delta lists rotate over 3 slots (phase mod 3): a CTA
// still applying phase G-1 must not see it overwritten by a CTA already in G+1.
__global__ void __launch_bounds__(kThreads, 1) pcd_wform_kernel(WformArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int2* L_rs = reinterpret_cast<int2*>(smem_raw);
    double* L_d = reinterpret_cast<double*>(smem_raw + kCap * sizeof(int2));
    double* D_d = reinterpret_cast<double*>(smem_raw);           // diag chunk: delta
    double* D_new = reinterpret_cast<double*>(smem_raw) + kCap;  // diag chunk: new value
    __shared__ int s_off[kMaxBlocks + 1];
    __shared__ int s_cnt;
    __shared__ double s_red[5][32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x, nblk = gridDim.x;
    const int p = a.p, m = a.m, w = a.w, w2 = a.w >> 1, half = a.half;
    const int c0 = b * w;
    const int wl = min(w, p - c0);
    const int c = c0 + tid;  // own column of a publisher thread (tid < wl)
    const int q_lo = min(b * a.share, half), q_hi = min(q_lo + a.share, half);
    double* __restrict__ Wb = a.W + (long long)b * a.slab;
    const double* __restrict__ Tb = a.T + (long long)b * a.slab;
    double* __restrict__ Ob = a.Om + (long long)b * a.slab;
    const unsigned long long nbu = (unsigned long long)nblk;
    unsigned long long epoch = 0;

    // ---- publish phase 0 of the first sweep, arrive
    if (tid < wl) {
        const int x = pub_row(0, c, m, p);
        if (x >= 0) a.pub[c] = make_double2(Wb[(long long)x * w + tid], Ob[(long long)x * w + tid]);
    }
    __syncthreads();
    bar_arrive(a.bar);
    if (b == 0 && tid == 0) a.rec_time[0] = globaltimer_ns();

    // ---- publisher state: cell (xp, c) for the next publish, prefetched value `pre`
    // (W after every phase before ph0), brought forward by phases ph0 (source row y0,
    // T[y0,c] = t0) and ph1 (y1, t1) at publish time.
    int xp = -1, ph0 = -1, y0 = -1, ph1 = 0, y1 = -1;
    double2 pre = make_double2(0.0, 0.0);
    double t0 = 0.0, t1 = 0.0;
    // prefetch for the publish done in phase `phA` (which publishes phase phA+1);
    // `phB` is the phase before phA, or -1 when nothing precedes it.
    auto prefetch = [&](int phB, int phA) {
        xp = -1;
        if (tid < wl) {
            const int phn = (phA == m) ? 0 : phA + 1;
            const int x = pub_row(phn, c, m, p);
            if (x >= 0) {
                xp = x;
                ph0 = phB;
                ph1 = phA;
                y0 = (phB >= 0) ? src_row(phB, x, m) : p;
                y1 = src_row(phA, x, m);
                pre = make_double2(Wb[(long long)x * w + tid], Ob[(long long)x * w + tid]);
                t0 = (y0 < p) ? __ldg(Tb + (long long)y0 * w + tid) : 0.0;
                t1 = (y1 < p) ? __ldg(Tb + (long long)y1 * w + tid) : 0.0;
            }
        }
    };
    prefetch(-1, 0);

    // optional phase profile (CONCORD_PHASE_PROFILE): CTA 0 / thread 0 clock64 per phase
    unsigned long long* prof = (a.prof && b == 0 && tid == 0) ? a.prof : nullptr;
    long long tmark = clock64();
#define PMARK(i)                                     \
    if (prof) {                                      \
        const long long t_ = clock64();              \
        prof[i] += (unsigned long long)(t_ - tmark); \
        tmark = t_;                                  \
    }

    int slot = 0;  // slot of the current phase; (slot+2)%3 is the previous one
    int it = 0, converged = 0;
    double smax = 0.0;  // max |delta| over this thread's share of the sweep
    int snnz = 0;
    while (true) {
        for (int ph = 0; ph <= m; ++ph) {
            bar_wait(a.bar, (++epoch) * nbu);
            PMARK(0);
            const int pslot = (slot == 0) ? 2 : slot - 1;
            const int nslot = (slot == 2) ? 0 : slot + 1;
            const double2* __restrict__ pb = a.pub + (size_t)slot * p;
            const double2* __restrict__ pbm = a.pub + (size_t)pslot * p;
            double2* __restrict__ pn = a.pub + (size_t)nslot * p;
            const bool diag = (ph == m);

            // ---- diagonal: convergence decision first (every CTA sees the same values)
            bool stop = false;
            double dmax_all = 0.0;
            if (diag) {
                double dm = 0.0;
                for (int i = tid; i < p; i += kThreads)
                    dm = fmax(dm, fabs(diag_delta(ldcg2(pb + i), __ldg(a.tdiag + i), a.n)));
                dm = warp_max(dm);
                if (lane == 0) s_red[0][warp] = dm;
                __syncthreads();
                const double off = __longlong_as_double((long long)__ldcg(a.rec_dmax + it));
                dmax_all = fmax(off, warp_max(lane < kThreads / 32 ? s_red[0][lane] : 0.0));
                stop = (dmax_all < a.delta_tol) || (it + 1 >= a.max_iter);
                __syncthreads();
            }

            // ---- publish phase ph+1
            if (!stop && xp >= 0) {
                double val = pre.x, om = pre.y, nv;
                if (y0 < p) {
                    const double d = row_delta(ph0, xp, y0, pbm, a.tdiag, m, a.shrink, a.n, nv);
                    if (d != 0.0) val = fma(d, t0, val);
                    if (y0 == c) om = nv;  // the correcting phase moved this very cell (only when m == 1)
                }
                if (y1 < p) {
                    const double d = row_delta(ph1, xp, y1, pb, a.tdiag, m, a.shrink, a.n, nv);
                    if (d != 0.0) val = fma(d, t1, val);
                    if (y1 == c) om = nv;
                }
                pn[c] = make_double2(val, om);
            }
            PMARK(1);

            // ---- share of the colour's closed forms -> list segment of this CTA
            if (!diag) {
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                const int c1 = m - 1 - ph;
                int2* seg_rs = a.list_rs + ((size_t)slot * nblk + b) * a.share;
                double2* seg_dn = a.list_dn + ((size_t)slot * nblk + b) * a.share;
                const int sid = kThreads - 1 - tid;  // share work starts on the last warps
                for (int base = q_lo; base < q_hi; base += kThreads) {
                    const int q = base + sid;
                    int r = 0, s = 0;
                    double d = 0.0, nv = 0.0;
                    if (q < q_hi) {
                        round_pair(q, m, c1, r, s);
                        if (s < p) {
                            d = pair_delta(ldcg2(pb + r), ldcg2(pb + s), __ldg(a.tdiag + r), __ldg(a.tdiag + s),
                                           a.shrink, nv);
                            if (d != 0.0) {
                                smax = fmax(smax, fabs(d));
                                ++snnz;
                            }
                        }
                    }
                    const unsigned mask = __ballot_sync(0xffffffffu, d != 0.0);
                    if (mask) {
                        int basepos = 0;
                        if (lane == 0) basepos = atomicAdd(&s_cnt, __popc(mask));
                        basepos = __shfl_sync(0xffffffffu, basepos, 0);
                        if (d != 0.0) {
                            const int at = basepos + __popc(mask & ((1u << lane) - 1u));
                            seg_rs[at] = make_int2(r, s);
                            seg_dn[at] = make_double2(d, nv);
                        }
                    }
                }
                __syncthreads();
                if (tid == 0) a.list_cnt[(size_t)slot * nblk + b] = s_cnt;
                if (ph == m - 1) {  // flush this sweep's share statistics
                    const double mw = warp_max(smax);
                    const double nw = warp_sum((double)snnz);
                    if (lane == 0) {
                        s_red[0][warp] = mw;
                        s_red[1][warp] = nw;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        const bool in = lane < kThreads / 32;
                        const double mb = warp_max(in ? s_red[0][lane] : 0.0);
                        const double nbk = warp_sum(in ? s_red[1][lane] : 0.0);
                        if (lane == 0) {
                            atomicMax(a.rec_dmax + it, (unsigned long long)__double_as_longlong(mb));
                            atomicAdd(reinterpret_cast<unsigned long long*>(a.rec_nnz + it),
                                      (unsigned long long)nbk);
                        }
                    }
                    smax = 0.0;
                    snnz = 0;
                }
            }
            PMARK(2);
            if (!stop) {
                __syncthreads();
                bar_arrive(a.bar);
            }

            // ---- apply the previous colour's non-zero deltas to the own slab
            const int prev = (ph == 0) ? -1 : ph - 1;  // phase 0 follows the diagonal (already applied)
            if (prev >= 0 && (it > 0 || ph > 0)) {
                for (int j = tid; j < nblk; j += kThreads) s_off[j] = __ldcg(a.list_cnt + (size_t)pslot * nblk + j);
                __syncthreads();
                if (warp == 0) {
                    int run = 0;
                    for (int j0 = 0; j0 < nblk; j0 += 32) {
                        const int j = j0 + lane;
                        int v = (j < nblk) ? s_off[j] : 0;
                        int incl = v;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int t = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += t;
                        }
                        if (j < nblk) s_off[j] = run + incl - v;
                        run += __shfl_sync(0xffffffffu, incl, 31);
                    }
                    if (lane == 0) s_off[nblk] = run;
                }
                __syncthreads();
                const int total = s_off[nblk];
                const int2* lrs = a.list_rs + (size_t)pslot * nblk * a.share;
                const double2* ldn = a.list_dn + (size_t)pslot * nblk * a.share;
                for (int e0 = 0; e0 < total; e0 += kCap) {
                    const int e1 = min(total, e0 + kCap);
                    for (int e = e0 + tid; e < e1; e += kThreads) {
                        int lo = 0, hi = nblk;  // segment: s_off[lo] <= e < s_off[lo+1]
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (s_off[mid] <= e) lo = mid;
                            else hi = mid;
                        }
                        const size_t at = (size_t)lo * a.share + (e - s_off[lo]);
                        const int2 rs = __ldcg(lrs + at);
                        const double2 dn = __ldcg(ldn + at);
                        if ((unsigned)(rs.y - c0) < (unsigned)wl) Ob[(long long)rs.x * w + (rs.y - c0)] = dn.y;
                        if ((unsigned)(rs.x - c0) < (unsigned)wl) Ob[(long long)rs.y * w + (rs.x - c0)] = dn.y;
                        L_rs[e - e0] = rs;
                        L_d[e - e0] = dn.x;
                    }
                    __syncthreads();
                    const int per = 2 * w2;
                    const int items = (e1 - e0) * per;
                    for (int base = 0; base < items; base += kThreads * kUnroll) {
                        double2 tv[kUnroll], wv[kUnroll];
                        double2* wp[kUnroll];
                        double dd[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int idx = base + u * kThreads + tid;
                            wp[u] = nullptr;
                            if (idx < items) {
                                const int e = idx / per;
                                const int rem = idx - e * per;
                                const int h = rem >= w2;
                                const int j2 = rem - h * w2;
                                const int2 rs = L_rs[e];
                                dd[u] = L_d[e];
                                const int dst = h ? rs.y : rs.x;
                                const int src = h ? rs.x : rs.y;
                                wp[u] = reinterpret_cast<double2*>(Wb + (long long)dst * w) + j2;
                                tv[u] = __ldg(reinterpret_cast<const double2*>(Tb + (long long)src * w) + j2);
                                wv[u] = *wp[u];
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            if (wp[u]) {
                                wv[u].x = fma(dd[u], tv[u].x, wv[u].x);
                                wv[u].y = fma(dd[u], tv[u].y, wv[u].y);
                                *wp[u] = wv[u];
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            PMARK(3);

            if (!diag) {
                prefetch(ph, ph + 1);
                PMARK(4);
                slot = nslot;
                continue;
            }

            // ---- diagonal step: prefetch (W before this phase), then the dense slab stream
            if (!stop) prefetch(m, 0);
            double q_acc = 0.0, pen_acc = 0.0, log_acc = 0.0;
            for (int i0 = 0; i0 < p; i0 += kCap) {
                const int iend = min(i0 + kCap, p);
                for (int i = i0 + tid; i < iend; i += kThreads) {
                    const double2 v = ldcg2(pb + i);
                    const double nv = diag_from_dot(v.x, v.y, __ldg(a.tdiag + i), a.n);
                    D_d[i - i0] = __dsub_rn(nv, v.y);
                    D_new[i - i0] = nv;
                }
                __syncthreads();
                const int items = (iend - i0) * w2;
                for (int base = 0; base < items; base += kThreads * kUnroll) {
                    double2 wv[kUnroll], tv[kUnroll], ov[kUnroll];
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        const int idx = base + u * kThreads + tid;
                        if (idx < items) {
                            const int ii = idx / w2;
                            const int j2 = idx - ii * w2;
                            const long long off = (long long)(i0 + ii) * w + 2 * j2;
                            wv[u] = *reinterpret_cast<const double2*>(Wb + off);
                            if (D_d[ii] != 0.0) tv[u] = __ldg(reinterpret_cast<const double2*>(Tb + off));
                            if (a.want_trace) ov[u] = *reinterpret_cast<const double2*>(Ob + off);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        const int idx = base + u * kThreads + tid;
                        if (idx < items) {
                            const int ii = idx / w2;
                            const int j2 = idx - ii * w2;
                            const int i = i0 + ii;
                            const long long off = (long long)i * w + 2 * j2;
                            const double d = D_d[ii];
                            if (d != 0.0) {
                                wv[u].x = fma(d, tv[u].x, wv[u].x);
                                wv[u].y = fma(d, tv[u].y, wv[u].y);
                                *reinterpret_cast<double2*>(Wb + off) = wv[u];
                            }
                            const int cj = c0 + 2 * j2;
                            const bool dg0 = (cj == i), dg1 = (cj + 1 == i);
                            if (a.want_trace) {
                                if (dg0 | dg1) {
                                    if (dg0) ov[u].x = D_new[ii];
                                    if (dg1) ov[u].y = D_new[ii];
                                    *reinterpret_cast<double2*>(Ob + off) = ov[u];
                                    log_acc += log(D_new[ii]);
                                }
                                q_acc = fma(wv[u].x, ov[u].x, q_acc);
                                q_acc = fma(wv[u].y, ov[u].y, q_acc);
                                if (i < cj) pen_acc += fabs(ov[u].x);
                                if (i < cj + 1) pen_acc += fabs(ov[u].y);
                            } else if (dg0 | dg1) {
                                Ob[off + (dg0 ? 0 : 1)] = D_new[ii];
                            }
                        }
                    }
                }
                __syncthreads();
            }
            ++it;
            PMARK(5);

            // ---- per-sweep records
            q_acc = warp_sum(q_acc);
            pen_acc = warp_sum(pen_acc);
            log_acc = warp_sum(log_acc);
            if (lane == 0) {
                s_red[1][warp] = q_acc;
                s_red[2][warp] = pen_acc;
                s_red[3][warp] = log_acc;
            }
            __syncthreads();
            if (warp == 0) {
                const bool in = lane < kThreads / 32;
                const double v1 = warp_sum(in ? s_red[1][lane] : 0.0);
                const double v2 = warp_sum(in ? s_red[2][lane] : 0.0);
                const double v3 = warp_sum(in ? s_red[3][lane] : 0.0);
                if (lane == 0) {
                    if (a.want_trace) {
                        double* ro = a.rec_obj + ((size_t)(it - 1) * nblk + b) * 3;
                        ro[0] = v1;
                        ro[1] = v2;
                        ro[2] = v3;
                    }
                    if (b == 0) {
                        a.rec_delta[it - 1] = dmax_all;
                        a.rec_time[it] = globaltimer_ns();
                    }
                }
            }
            __syncthreads();
            PMARK(6);
            if (stop) {
                converged = dmax_all < a.delta_tol;
                break;
            }
            slot = nslot;
        }
        if (it > 0 && (converged || it >= a.max_iter)) break;
    }
#undef PMARK
    if (b == 0 && tid == 0) {
        a.status[0] = it;
        a.status[1] = converged;
    }
}

// --------------------------------------------------------------- layout kernels
// Row-major p x p (leading dim ld) -> slab-major (zero padding).
__global__ void pack_slabs_kernel(const double* __restrict__ src, long long ld, double* __restrict__ dst,
                                  int p, int w, int nblk) {
    const long long total = (long long)nblk * p * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / ((long long)p * w);
        const long long rem = e - b * p * w;
        const int i = (int)(rem / w);
        const int j = (int)(rem - (long long)i * w);
        const long long c = b * w + j;
        dst[e] = (c < p) ? src[(long long)i * ld + c] : 0.0;
    }
}

// Slab-major -> row-major p x p.
__global__ void unpack_slabs_kernel(const double* __restrict__ src, double* __restrict__ dst, int p, int w) {
    const long long total = (long long)p * p;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / p);
        const int c = (int)(e - (long long)i * p);
        const int b = c / w;
        dst[e] = src[(long long)b * p * w + (long long)i * w + (c - b * w)];
    }
}

__global__ void slab_diag_kernel(const double* __restrict__ slab, double* __restrict__ diag, int p, int w) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
        const int b = i / w;
        diag[i] = slab[(long long)b * p * w + (long long)i * w + (i - b * w)];
    }
}

__global__ void slab_set_identity_kernel(double* __restrict__ slab, int p, int w) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
        const int b = i / w;
        slab[(long long)b * p * w + (long long)i * w + (i - b * w)] = 1.0;
    }
}

// Count exact non-zeros of the strict upper triangle (model.py:249-253).
__global__ void slab_edge_count_kernel(const double* __restrict__ slab, int p, int w, int nblk,
                                       unsigned long long* __restrict__ out) {
    unsigned long long local = 0;
    const long long total = (long long)nblk * p * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / ((long long)p * w);
        const long long rem = e - b * p * w;
        const int i = (int)(rem / w);
        const long long c = b * w + (rem - (long long)i * w);
        if (c < p && i < c && slab[e] != 0.0) ++local;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

// W (slab) = Omega_init * T for a warm start, from a CSR copy of Omega_init.
// Row i of W is sum_k om[i,k] T[k,:]; each block streams its own slab.
__global__ void wform_init_csr_kernel(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                                      const double* __restrict__ vals, const double* __restrict__ Tslab,
                                      double* __restrict__ Wslab, int p, int w) {
    const int b = blockIdx.y;
    const double* Tb = Tslab + (long long)b * p * w;
    double* Wb = Wslab + (long long)b * p * w;
    const int w2 = w >> 1;
    const long long items = (long long)p * w2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < items;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / w2);
        const int j2 = (int)(idx - (long long)i * w2);
        double2 acc = make_double2(0.0, 0.0);
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const double v = vals[e];
            const double2 tv = __ldg(reinterpret_cast<const double2*>(Tb + (long long)colidx[e] * w) + j2);
            acc.x = fma(v, tv.x, acc.x);
            acc.y = fma(v, tv.y, acc.y);
        }
        reinterpret_cast<double2*>(Wb + (long long)i * w)[j2] = acc;
    }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_pcd_wform(const WformArgs& args, int nblk, cudaStream_t st) {
    const size_t smem = wform_smem_bytes(args.w);
    cudaError_t e = cudaFuncSetAttribute(pcd_wform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    WformArgs copy = args;
    void* kargs[] = {&copy};
    return cudaLaunchCooperativeKernel((void*)pcd_wform_kernel, dim3(nblk), dim3(kThreads), kargs, smem, st);
}

cudaError_t wform_max_blocks(int w, int* max_blocks) {
    const size_t smem = wform_smem_bytes(w);
    cudaError_t e = cudaFuncSetAttribute(pcd_wform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcd_wform_kernel, kThreads, smem);
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

cudaError_t launch_pack_slabs(const double* src, long long ld, double* dst, int p, int w, int nblk,
                              cudaStream_t st) {
    pack_slabs_kernel<<<grid_for((long long)nblk * p * w), 256, 0, st>>>(src, ld, dst, p, w, nblk);
    return cudaGetLastError();
}

cudaError_t launch_unpack_slabs(const double* src, double* dst, int p, int w, cudaStream_t st) {
    unpack_slabs_kernel<<<grid_for((long long)p * p), 256, 0, st>>>(src, dst, p, w);
    return cudaGetLastError();
}

cudaError_t launch_slab_diag(const double* slab, double* diag, int p, int w, cudaStream_t st) {
    slab_diag_kernel<<<grid_for(p), 256, 0, st>>>(slab, diag, p, w);
    return cudaGetLastError();
}

cudaError_t launch_slab_identity(double* slab, int p, int w, int nblk, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(slab, 0, sizeof(double) * (size_t)nblk * p * w, st);
    if (e != cudaSuccess) return e;
    slab_set_identity_kernel<<<grid_for(p), 256, 0, st>>>(slab, p, w);
    return cudaGetLastError();
}

cudaError_t launch_slab_edge_count(const double* slab, int p, int w, int nblk, unsigned long long* out,
                                   cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    slab_edge_count_kernel<<<grid_for((long long)nblk * p * w), 256, 0, st>>>(slab, p, w, nblk, out);
    return cudaGetLastError();
}

cudaError_t launch_wform_init_csr(const int* rowptr, const int* colidx, const double* vals, const double* Tslab,
                                  double* Wslab, int p, int w, int nblk, cudaStream_t st) {
    long long items = (long long)p * (w >> 1);
    int gx = (int)((items + 255) / 256);
    if (gx > 64) gx = 64;
    wform_init_csr_kernel<<<dim3(gx, nblk), 256, 0, st>>>(rowptr, colidx, vals, Tslab, Wslab, p, w);
    return cudaGetLastError();
}

}  // namespace concord
