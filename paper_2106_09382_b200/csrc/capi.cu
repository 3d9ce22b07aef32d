// extern "C" ABI of libconcord_b200.so (include/concord_pcd.h).
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/concord_pcd.h"
#include "pcd_wform.h"

using namespace concord;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            (void)cudaGetLastError(); /* reported here, not again by the next launch check */      \
            return fail(_e == cudaErrorMemoryAllocation ? CONCORD_ERR_OOM : CONCORD_ERR_CUDA,      \
                        "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e));        \
        }                                                                                          \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename T>
cudaError_t dalloc(T** ptr, size_t count) {
    *ptr = nullptr;
    if (count == 0) count = 1;
    const cudaError_t e = cudaMalloc((void**)ptr, sizeof(T) * count);
    // a failed allocation also sets the runtime's last error, which the next kernel launch's
    // cudaGetLastError() would report as its own failure: the caller gets the error here instead
    if (e != cudaSuccess) (void)cudaGetLastError();
    return e;
}

int check_device(int32_t device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(CONCORD_ERR_NO_DEVICE, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(CONCORD_ERR_ARG, "device %d out of range [0,%d)", device, count);
    return CONCORD_OK;
}

// Byte offsets of the exchange buffers inside one arena (identical on every shard).
struct ArenaLayout {
    size_t pub, dring, list_rs, list_dn, list_cnt, bar, dmax;
    // the blocked kernel's exchange buffers (pcd_qblock.cu), present when qb_sr > 0
    size_t qb_stW, qb_stO, qb_stT, qb_diagv, qb_dring, qb_lrs, qb_ldn, qb_lcnt;
    size_t bytes;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

ArenaLayout arena_layout(int p, int rd, int rl, int nblk_tot, int share, int qb_sr = 0, int qb_rd = 0,
                         int qb_rl = 0) {
    ArenaLayout L{};
    size_t o = 0;
    L.pub = o;
    o = align256(o + sizeof(double2) * 3 * (size_t)p);
    L.dring = o;
    o = align256(o + sizeof(double) * (size_t)rd * p);
    L.list_rs = o;
    o = align256(o + sizeof(int2) * (size_t)rl * nblk_tot * share);
    L.list_dn = o;
    o = align256(o + sizeof(double2) * (size_t)rl * nblk_tot * share);
    L.list_cnt = o;
    o = align256(o + sizeof(int) * (size_t)rl * nblk_tot);
    L.bar = o;
    o = align256(o + sizeof(unsigned long long));
    L.dmax = o;  // [WFORM_DMAX_RING] max |delta| per sweep, then [WFORM_DMAX_RING] yield words (blocked kernel)
    o = align256(o + sizeof(unsigned long long) * 2 * WFORM_DMAX_RING);
    if (qb_sr > 0) {
        L.qb_stW = o;
        o = align256(o + sizeof(double) * (size_t)qb_sr * p);
        L.qb_stO = o;
        o = align256(o + sizeof(double) * (size_t)qb_sr * p);
        L.qb_stT = o;
        o = align256(o + sizeof(double) * (size_t)qb_sr * (QB_DMAX - 1) * p);
        L.qb_diagv = o;
        o = align256(o + sizeof(double2) * (size_t)p);
        L.qb_dring = o;
        o = align256(o + sizeof(double) * (size_t)qb_rd * p);
        L.qb_lrs = o;
        o = align256(o + sizeof(int2) * (size_t)qb_rl * nblk_tot * share);
        L.qb_ldn = o;
        o = align256(o + sizeof(double2) * (size_t)qb_rl * nblk_tot * share);
        L.qb_lcnt = o;
        o = align256(o + sizeof(int) * (size_t)qb_rl * nblk_tot);
    }
    L.bytes = o;
    return L;
}

}  // namespace

struct concord_solver {
    int dev = 0;
    int p = 0;
    int w = 0;
    int G = 1;            // shards
    int rank = -1;        // -1: every shard on this device; else the one shard this process owns
    int nblk_loc = 0;     // slabs per shard
    int nblk_tot = 0;     // slabs over all shards
    int blk0 = 0;         // first global slab of this solver's launch
    int nblk_launch = 0;  // slabs (CTAs) this solver launches
    long long slab = 0;
    int lmax = 1, rd = 0, rl = 0, share = 0, nsh = 0;
    bool qb = false;       // temporally blocked chain (pcd_qblock.cu)
    int qb_D = 0, qb_NB = 0, qb_sr = 0, qb_rd = 0, qb_rl = 0;
    int qb_nbuf = 1, qb_td = 0, qb_ring = 6;  // shared-memory plan of the blocked kernel
    int qb_cw = QB_CHAIN_WARPS;               // its chain-warp variant (4, 6, 8)
    double* Tfull = nullptr;  // process shard on the blocked kernel: every slab of T (the cells' T entries)
    // storage of W, T, Om: local slab b, row i, slab column j at b * ss + i * ld + j.  Row-major
    // (ss = w, ld = the launch's columns) for the blocked kernel -- every CTA streams the same
    // rows at the same time, so each row is one contiguous DRAM stretch; slab layout (ss = p*w,
    // ld = w) for the per-phase kernel.  ssT / ldT: the same for Tfull.
    long long ss = 0, ld = 0, ssT = 0, ldT = 0;
    long long* hang = nullptr;  // mapped host memory: the fit kernels' watchdog report
    volatile int* yield = nullptr;  // mapped host flag: the running blocked fit stops at its next sweep end
    bool resume = false;            // the next fit continues from an imported (Omega, W) state
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    double* T = nullptr;
    double* W = nullptr;
    double* Om = nullptr;
    double* tdiag = nullptr;
    double* stage = nullptr;  // p x p row-major scratch (lazy)
    double2* diagd = nullptr;
    ArenaLayout L{};
    void* arena[WFORM_MAX_SHARDS] = {};
    bool arena_owned[WFORM_MAX_SHARDS] = {};
    bool peers_open = false;
    unsigned long long bar_base = 0;  // barrier arrivals so far (identical on every shard)
    int it_base = 0;                  // sweeps run so far (identical on every shard)
    unsigned long long* edges = nullptr;
    int* status = nullptr;
    double* rec_delta = nullptr;
    double* rec_obj = nullptr;
    unsigned long long* rec_time = nullptr;
    long long* rec_nnz = nullptr;
    int rec_cap = 0;
    int last_iters = 0;
    long long* csr_rowptr = nullptr;  // int64: a dense init at p >= 46341 has > 2^31 entries
    int* csr_col = nullptr;
    double* csr_val = nullptr;
    long long csr_cap = 0;
    double n = 0.0;
    bool have_gram = false;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
};

namespace {

int ensure_stage(concord_solver* s) {
    if (!s->stage) CK(dalloc(&s->stage, (size_t)s->p * s->p));
    return CONCORD_OK;
}

int ensure_records(concord_solver* s, int cap) {
    if (cap <= s->rec_cap) return CONCORD_OK;
    cudaFree(s->rec_delta);
    cudaFree(s->rec_obj);
    cudaFree(s->rec_time);
    cudaFree(s->rec_nnz);
    s->rec_delta = nullptr;
    s->rec_obj = nullptr;
    s->rec_time = nullptr;
    s->rec_nnz = nullptr;
    CK(dalloc(&s->rec_delta, cap));
    CK(dalloc(&s->rec_nnz, cap));
    CK(dalloc(&s->rec_obj, (size_t)cap * s->nblk_launch * 3));
    CK(dalloc(&s->rec_time, cap + 1));
    s->rec_cap = cap;
    return CONCORD_OK;
}

int ncols_local(const concord_solver* s) {
    const int c0 = s->blk0 * s->w;
    const int c1 = (s->blk0 + s->nblk_launch) * s->w;
    return (c1 < s->p ? c1 : s->p) - (c0 < s->p ? c0 : s->p);
}

// Row-major p x p (host or device) -> this solver's T slabs and the replicated diagonal.
int set_gram_rowmajor(concord_solver* s, const double* src, int32_t where) {
    const double* dsrc = src;
    if (where == CONCORD_HOST) {
        int rc = ensure_stage(s);
        if (rc) return rc;
        CK(cudaMemcpyAsync(s->stage, src, sizeof(double) * (size_t)s->p * s->p, cudaMemcpyHostToDevice,
                           s->stream));
        dsrc = s->stage;
    }
    CK(launch_pack_slabs(dsrc, s->p, s->T, s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->stream));
    if (s->Tfull)
        CK(launch_pack_slabs(dsrc, s->p, s->Tfull, s->p, s->w, s->ssT, s->ldT, s->nblk_tot, 0, s->stream));
    CK(launch_rowmajor_diag(dsrc, s->tdiag, s->p, s->stream));
    std::vector<double> d(s->p);
    CK(cudaMemcpyAsync(d.data(), s->tdiag, sizeof(double) * s->p, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (int i = 0; i < s->p; ++i)
        if (!(d[i] > 0.0)) {
            s->have_gram = false;
            return fail(CONCORD_ERR_ZERO_VARIANCE, "column %d has zero sum of squares", i);
        }
    s->have_gram = true;
    return CONCORD_OK;
}

int download_slabs(concord_solver* s, const double* src, double* out, int32_t where) {
    if (where == CONCORD_DEVICE) {
        CK(launch_unpack_slabs(src, out, s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        return CONCORD_OK;
    }
    int rc = ensure_stage(s);
    if (rc) return rc;
    CK(launch_unpack_slabs(src, s->stage, s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->stream));
    CK(cudaMemcpyAsync(out, s->stage, sizeof(double) * (size_t)s->p * ncols_local(s), cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return CONCORD_OK;
}

// Warm start: Omega slabs from omega_init, W = Omega_init * T through a CSR copy.
int init_warm(concord_solver* s, const double* om, int32_t where) {
    const int p = s->p;
    std::vector<double> host;
    const double* h = om;
    if (where == CONCORD_DEVICE) {
        host.resize((size_t)p * p);
        CK(cudaMemcpyAsync(host.data(), om, sizeof(double) * (size_t)p * p, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        h = host.data();
    }
    std::vector<long long> rowptr(p + 1, 0);
    std::vector<int> col;
    std::vector<double> val;
    for (int i = 0; i < p; ++i) {
        const double* row = h + (size_t)i * p;
        for (int j = 0; j < p; ++j)
            if (row[j] != 0.0) {
                col.push_back(j);
                val.push_back(row[j]);
            }
        rowptr[i + 1] = (long long)col.size();
    }
    const long long nnz = (long long)col.size();
    if (nnz > s->csr_cap) {
        cudaFree(s->csr_col);
        cudaFree(s->csr_val);
        s->csr_col = nullptr;
        s->csr_val = nullptr;
        CK(dalloc(&s->csr_col, nnz));
        CK(dalloc(&s->csr_val, nnz));
        s->csr_cap = nnz;
    }
    if (!s->csr_rowptr) CK(dalloc(&s->csr_rowptr, p + 1));
    CK(cudaMemcpyAsync(s->csr_rowptr, rowptr.data(), sizeof(long long) * (p + 1), cudaMemcpyHostToDevice, s->stream));
    if (nnz) {
        CK(cudaMemcpyAsync(s->csr_col, col.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice, s->stream));
        CK(cudaMemcpyAsync(s->csr_val, val.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, s->stream));
    }
    int rc = ensure_stage(s);
    if (rc) return rc;
    CK(cudaMemcpyAsync(s->stage, h, sizeof(double) * (size_t)p * p, cudaMemcpyHostToDevice, s->stream));
    CK(launch_pack_slabs(s->stage, p, s->Om, p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->stream));
    CK(launch_wform_init_csr(s->csr_rowptr, s->csr_col, s->csr_val, s->T, s->W, p, s->w, s->ss, s->ld, s->nblk_launch,
                             s->stream));
    CK(cudaStreamSynchronize(s->stream));  // host vectors go out of scope
    return CONCORD_OK;
}

WformCopies copies(const concord_solver* s) {
    WformCopies x;
    memset(&x, 0, sizeof(x));
    for (int r = 0; r < s->G; ++r) {
        char* base = static_cast<char*>(s->arena[r]);
        x.pub[r] = reinterpret_cast<double2*>(base + s->L.pub);
        x.dring[r] = reinterpret_cast<double*>(base + s->L.dring);
        x.list_rs[r] = reinterpret_cast<int2*>(base + s->L.list_rs);
        x.list_dn[r] = reinterpret_cast<double2*>(base + s->L.list_dn);
        x.list_cnt[r] = reinterpret_cast<int*>(base + s->L.list_cnt);
        x.bar[r] = reinterpret_cast<unsigned long long*>(base + s->L.bar);
        x.dmax[r] = reinterpret_cast<unsigned long long*>(base + s->L.dmax);
    }
    return x;
}

// Shared-memory plan of the blocked kernel for p (slabs of a default single-device layout:
// nblk CTAs, `share` pairs each), first that fits 227 KB, in order of value: two cell buffers
// (the next block's cells built during the colours -- only useful while the prefetch group, the
// chain warps the colours leave free, has at most ~5 cells per thread; beyond that part A
// outlasts the colours, measured at p=20000), the T diagonal in shared memory, the deepest
// cp.async row ring.  Returns false when nothing fits (the per-phase kernel then runs).
struct QbPlan {
    int D, nbuf, td, ring;
    size_t smem;
};
static bool qblock_plan(int p, int nblk, int share, int D, bool allow_overlap, int chain_warps, QbPlan* out) {
    const int m = p + (p & 1) - 1;
    if (D < 2) D = 2;
    if (D > QB_DMAX) D = QB_DMAX;
    if (2 * D > m + 1) D = (m + 1) / 2;
    int cw = qblock_colour_warps(chain_warps, share, D);
    if (const char* e = getenv("CONCORD_QB_CW")) {  // tuning: a negative value fixes the colour group's warps
        const int v = atoi(e);
        cw = v < 0 ? -v : (v > cw ? v : cw);
    }
    int pf_cells = 5;  // part A overlaps the colours when the prefetch group has at most this many cells per thread
    if (const char* e = getenv("CONCORD_QB_PF_CELLS")) pf_cells = atoi(e);
    const int pf_threads = 32 * (chain_warps - cw);
    const bool can_overlap = allow_overlap && pf_threads > 0 && qblock_cellcap(share, D) <= pf_cells * pf_threads;
    static const int plans[][3] = {{2, 1, 6}, {2, 0, 6}, {1, 1, 6}, {1, 0, 6}, {1, 0, 4}, {1, 0, 2}};
    const int td_ok = wform_tdiag_in_smem(p);
    for (const auto& pl : plans) {
        if (pl[0] == 2 && !can_overlap) continue;
        if (pl[1] && !td_ok) continue;
        const size_t smem = qblock_smem_bytes(chain_warps, p, nblk, share, D, pl[1], pl[0], pl[2]);
        if (smem + 2048 <= 227 * 1024) {  // + static shared memory
            *out = QbPlan{D, pl[0], pl[1], pl[2], smem};
            return true;
        }
    }
    return false;
}

// Plan of the temporally blocked chain (pcd_qblock.cu); leaves s->qb false when it does not fit.
// Its exchange buffers are carved from the shard arenas (arena_layout) by create_common.
int setup_qblock(concord_solver* s) {
    const int p = s->p;
    const int m = p + (p & 1) - 1;
    int D = QB_DEFAULT_D;
    if (const char* e = getenv("CONCORD_QB_D")) D = atoi(e);
    bool allow_overlap = true;
    if (const char* e = getenv("CONCORD_QB_NBUF")) allow_overlap = atoi(e) >= 2;
    QbPlan plan;
    if (!qblock_plan(p, s->nblk_tot, s->share, D, allow_overlap, s->qb_cw, &plan)) return CONCORD_OK;  // per-phase kernel
    D = plan.D;
    s->qb_nbuf = plan.nbuf;
    s->qb_td = plan.td;
    s->qb_ring = plan.ring;
    if (const char* e = getenv("CONCORD_QB_RING")) {  // tuning: a deeper ring when it still fits
        const int r = atoi(e);
        if ((r == 2 || r == 4 || r == 6 || r == 8) &&
            qblock_smem_bytes(s->qb_cw, p, s->nblk_tot, s->share, plan.D, plan.td, plan.nbuf, r) + 2048 <= 227 * 1024)
            s->qb_ring = r;
    }
    s->qb_D = D;
    CK(qblock_reserve_smem(s->qb_cw, qblock_smem_bytes(s->qb_cw, p, s->nblk_tot, s->share, D, s->qb_td, s->qb_nbuf,
                                                        s->qb_ring)));
    s->qb_NB = (m + 1 + D - 1) / D;
    s->qb_sr = 4 * D + 4;
    s->qb_rd = 8 * D + 8;
    s->qb_rl = 10 * D + 8;
    s->qb = true;
    return CONCORD_OK;
}

// Common constructor: G shards of nblk_loc slabs; rank < 0 keeps every shard on `device`.
int create_common(int64_t p, int32_t device, int32_t n_blocks, int32_t n_shards, int32_t rank,
                  concord_solver** out) {
    if (!out) return fail(CONCORD_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (p < 2) return fail(CONCORD_ERR_ARG, "T must be square with p >= 2, got p=%lld", (long long)p);
    if (p > (1LL << 30)) return fail(CONCORD_ERR_ARG, "p=%lld too large", (long long)p);
    if (n_shards < 1 || n_shards > WFORM_MAX_SHARDS)
        return fail(CONCORD_ERR_ARG, "n_shards=%d outside [1,%d]", n_shards, WFORM_MAX_SHARDS);
    if (rank >= n_shards) return fail(CONCORD_ERR_ARG, "rank %d >= n_shards %d", rank, n_shards);
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const int ip = (int)p;
    const int G = n_shards;
    // CTAs one launch may use: all shards share the device when rank < 0
    int w;
    if (n_blocks > 0) {
        w = (ip + n_blocks - 1) / n_blocks;
    } else {
        const int tot = (rank < 0) ? nsm : nsm * G;
        w = (ip + tot - 1) / tot;
        if (w < 8) w = 8;
    }
    w = (w + 1) & ~1;
    if (n_blocks <= 0) {
        // default layout: rows of w doubles on whole 32-byte sectors (w a multiple of 4) when that
        // keeps >= 90% of the slabs -- the random row streams then move no partial sectors (p=5000
        // on 148 SMs: w=34 -> 36 on 139 slabs, the dense lambda=0.1 fit 1.93 -> 1.70 s, the sparse
        // lambda=0.3 fit 0.25 -> 0.26 s; profiles/r02/align.log).  An explicit slab count (a lane of
        // PathScheduler, mostly sparse fits) keeps its width: there 122 -> 124 cost the sparse fits 8%.
        const int w4 = (w + 3) & ~3;
        const int need = (ip + w - 1) / w, need4 = (ip + w4 - 1) / w4;
        if (w4 != w && 10 * need4 >= 9 * need) w = w4;
    }
    int nblk_loc = 0;
    for (;;) {
        if (w > 4096) return fail(CONCORD_ERR_ARG, "p=%d needs slab width %d (too wide)", ip, w);
        const int need = (ip + w - 1) / w;
        nblk_loc = (need + G - 1) / G;
        int max_blocks = 0;
        CK(wform_max_blocks(w, ip, nblk_loc * G, &max_blocks));
        const int launch = (rank < 0) ? nblk_loc * G : nblk_loc;
        if (launch <= max_blocks && nblk_loc * G <= WFORM_MAX_BLOCKS) break;
        w += 2;
    }
    concord_solver* s = new concord_solver();
    s->dev = device;
    s->p = ip;
    s->w = w;
    s->G = G;
    s->rank = rank;
    s->nblk_loc = nblk_loc;
    s->nblk_tot = nblk_loc * G;
    s->blk0 = (rank < 0) ? 0 : rank * nblk_loc;
    s->nblk_launch = (rank < 0) ? s->nblk_tot : nblk_loc;
    s->slab = (long long)ip * w;
    const size_t tot = (size_t)s->nblk_launch * s->slab;
    auto cleanup = [&](int code) {
        concord_solver_destroy(s);
        return code;
    };
#define CKC(expr)                                                                                  \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess && ((void)cudaGetLastError(), true))                                 \
            return cleanup(fail(_e == cudaErrorMemoryAllocation ? CONCORD_ERR_OOM : CONCORD_ERR_CUDA, \
                                "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e))); \
    } while (0)
    CKC(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking));
    s->stream = s->own_stream;
    CKC(dalloc(&s->T, tot));
    CKC(dalloc(&s->W, tot));
    CKC(dalloc(&s->Om, tot));
    CKC(cudaMemsetAsync(s->T, 0, sizeof(double) * tot, s->stream));
    CKC(cudaMemsetAsync(s->W, 0, sizeof(double) * tot, s->stream));
    CKC(cudaMemsetAsync(s->Om, 0, sizeof(double) * tot, s->stream));
    CKC(cudaHostAlloc((void**)&s->hang, 8 * sizeof(long long), cudaHostAllocMapped));
    memset(s->hang, 0, 8 * sizeof(long long));
    CKC(cudaHostAlloc((void**)&s->yield, sizeof(int), cudaHostAllocMapped));
    s->yield[0] = 0;
    CKC(dalloc(&s->tdiag, ip));
    CKC(dalloc(&s->diagd, (size_t)s->nblk_launch * ip));
    {
        const int half = (ip + (ip & 1)) / 2;
        int share_min = WFORM_SHARE_MIN;
        if (const char* e = getenv("CONCORD_SHARE_MIN")) share_min = atoi(e);
        s->share = (half + s->nblk_tot - 1) / s->nblk_tot;
        if (s->share < share_min) s->share = share_min < half ? share_min : half;
        s->nsh = (half + s->share - 1) / s->share;
        s->lmax = wform_lag_cap(w, 2 * half - 1);
        s->rd = s->lmax + 3;
        s->rl = s->lmax + 4;
    }
    // the temporally blocked kernel (default for p >= 256, every shard layout); CONCORD_KERNEL=wform
    // selects the per-phase one
    {
        bool use_qb = ip >= 256;
        if (const char* e = getenv("CONCORD_KERNEL")) use_qb = use_qb && strcmp(e, "qblock") == 0;
        else use_qb = use_qb && QB_DEFAULT;
        if (use_qb) {
            const int rc = setup_qblock(s);
            if (rc) return cleanup(rc);
        }
        s->L = s->qb ? arena_layout(ip, s->rd, s->rl, s->nblk_tot, s->share, s->qb_sr, s->qb_rd, s->qb_rl)
                     : arena_layout(ip, s->rd, s->rl, s->nblk_tot, s->share);
        // row-major storage for the blocked kernel (32-bit double2 row offsets: p * columns / 2 < 2^31)
        bool rowmajor = s->qb && (long long)ip * s->nblk_tot * w / 2 < (1LL << 31);
        if (const char* e = getenv("CONCORD_LAYOUT")) rowmajor = rowmajor && strcmp(e, "slab") != 0;
        s->ss = rowmajor ? w : s->slab;
        s->ld = rowmajor ? (long long)s->nblk_launch * w : w;
        s->ssT = rowmajor ? w : s->slab;
        s->ldT = rowmajor ? (long long)s->nblk_tot * w : w;
    }
    for (int r = 0; r < G; ++r) {
        if (rank >= 0 && r != rank) continue;  // peers' arenas are opened by concord_shard_open_peers
        CKC(cudaMalloc(&s->arena[r], s->L.bytes));
        s->arena_owned[r] = true;
        CKC(cudaMemsetAsync(s->arena[r], 0, s->L.bytes, s->stream));
    }
    s->peers_open = (rank < 0) || G == 1;
    CKC(dalloc(&s->edges, 1));
    CKC(dalloc(&s->status, 2));
    for (auto& e : s->ev) CKC(cudaEventCreate(&e));
    if (s->qb && rank >= 0 && G > 1) {  // the cells read T entries of every column
        CKC(dalloc(&s->Tfull, (size_t)s->nblk_tot * s->slab));
        CKC(cudaMemsetAsync(s->Tfull, 0, sizeof(double) * (size_t)s->nblk_tot * s->slab, s->stream));
    }
    CKC(cudaStreamSynchronize(s->stream));
#undef CKC
    *out = s;
    return CONCORD_OK;
}

}  // namespace

extern "C" {

int concord_abi_version(void) { return CONCORD_ABI_VERSION; }

const char* concord_last_error(void) { return g_err.c_str(); }

int concord_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) c = 0;
    if (count) *count = c;
    return CONCORD_OK;
}

int concord_solver_create(int64_t p, int32_t device, int32_t n_blocks, concord_solver** out) {
    return create_common(p, device, n_blocks, 1, -1, out);
}

int concord_solver_create_sharded(int64_t p, int32_t device, int32_t n_blocks, int32_t n_shards,
                                  concord_solver** out) {
    return create_common(p, device, n_blocks, n_shards, -1, out);
}

int concord_shard_create(int64_t p, int32_t n_shards, int32_t rank, int32_t device, int32_t n_blocks,
                         concord_solver** out) {
    if (rank < 0) return fail(CONCORD_ERR_ARG, "rank must be >= 0");
    return create_common(p, device, n_blocks, n_shards, rank, out);
}

int concord_shard_ipc_handle(concord_solver* s, void* handle_out) {
    if (!s || !handle_out) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (s->rank < 0) return fail(CONCORD_ERR_ARG, "not a process shard");
    DeviceGuard g(s->dev);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, s->arena[s->rank]));
    static_assert(sizeof(cudaIpcMemHandle_t) <= CONCORD_SHARD_HANDLE_BYTES, "handle size");
    memset(handle_out, 0, CONCORD_SHARD_HANDLE_BYTES);
    memcpy(handle_out, &h, sizeof(h));
    return CONCORD_OK;
}

int concord_shard_open_peers(concord_solver* s, const void* handles) {
    if (!s || !handles) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (s->rank < 0) return fail(CONCORD_ERR_ARG, "not a process shard");
    DeviceGuard g(s->dev);
    const unsigned char* hb = static_cast<const unsigned char*>(handles);
    for (int r = 0; r < s->G; ++r) {
        if (r == s->rank || s->arena[r]) continue;
        cudaIpcMemHandle_t h;
        memcpy(&h, hb + (size_t)r * CONCORD_SHARD_HANDLE_BYTES, sizeof(h));
        CK(cudaIpcOpenMemHandle(&s->arena[r], h, cudaIpcMemLazyEnablePeerAccess));
        s->arena_owned[r] = false;
    }
    s->peers_open = true;
    return CONCORD_OK;
}

int concord_solver_set_chain_warps(concord_solver* s, int32_t chain_warps) {
    if (!s) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (!qblock_variant_ok(chain_warps)) return fail(CONCORD_ERR_ARG, "chain_warps must be 4, 6 or 8, got %d", chain_warps);
    if (!s->qb) return CONCORD_OK;  // the per-phase kernel has one variant
    const int keep = s->qb_cw;
    s->qb_cw = chain_warps;
    const int rc = setup_qblock(s);  // re-plans shared memory for the variant (buffers do not change)
    if (rc || !s->qb) {
        s->qb_cw = keep;
        s->qb = true;
        setup_qblock(s);
        return rc ? rc : fail(CONCORD_ERR_ARG, "variant with %d chain warps does not fit shared memory", chain_warps);
    }
    return CONCORD_OK;
}

int concord_solver_request_yield(concord_solver* s, int32_t on) {
    if (!s || !s->yield) return fail(CONCORD_ERR_ARG, "solver is NULL");
    s->yield[0] = on ? 1 : 0;
    return CONCORD_OK;
}

int concord_solver_export_state(concord_solver* s, double* omega_out, double* w_out, int32_t where) {
    if (!s || !omega_out || !w_out) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (s->G > 1 || s->rank >= 0) return fail(CONCORD_ERR_ARG, "state export needs an unsharded solver");
    DeviceGuard g(s->dev);
    int rc = download_slabs(s, s->Om, omega_out, where);
    if (rc) return rc;
    return download_slabs(s, s->W, w_out, where);
}

int concord_solver_import_state(concord_solver* s, const double* omega, const double* w, int32_t where) {
    if (!s || !omega || !w) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (s->G > 1 || s->rank >= 0) return fail(CONCORD_ERR_ARG, "state import needs an unsharded solver");
    if (!s->have_gram) return fail(CONCORD_ERR_ARG, "no Gram matrix set");
    DeviceGuard g(s->dev);
    const size_t bytes = sizeof(double) * (size_t)s->p * s->p;
    const double* src[2] = {omega, w};
    double* dst[2] = {s->Om, s->W};
    for (int k = 0; k < 2; ++k) {
        const double* d = src[k];
        if (where == CONCORD_HOST) {
            int rc = ensure_stage(s);
            if (rc) return rc;
            CK(cudaMemcpyAsync(s->stage, src[k], bytes, cudaMemcpyHostToDevice, s->stream));
            d = s->stage;
        }
        CK(cudaMemsetAsync(dst[k], 0, sizeof(double) * (size_t)s->nblk_launch * s->slab, s->stream));
        CK(launch_pack_slabs(d, s->p, dst[k], s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->stream));
    }
    CK(cudaStreamSynchronize(s->stream));
    s->resume = true;
    return CONCORD_OK;
}

int concord_solver_reserve(concord_solver* s, int32_t max_iter) {
    if (!s) return fail(CONCORD_ERR_ARG, "solver is NULL");
    if (max_iter < 1) return fail(CONCORD_ERR_ARG, "max_iter must be at least 1");
    DeviceGuard g(s->dev);
    int rc = ensure_stage(s);
    if (rc) return rc;
    return ensure_records(s, max_iter);
}

int concord_solver_copy_gram(concord_solver* dst, concord_solver* src) {
    if (!dst || !src) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (dst == src) return fail(CONCORD_ERR_ARG, "source and destination are the same solver");
    if (dst->p != src->p || dst->dev != src->dev) return fail(CONCORD_ERR_ARG, "solvers differ in p or device");
    if (dst->G > 1 || dst->rank >= 0 || src->G > 1 || src->rank >= 0)
        return fail(CONCORD_ERR_ARG, "Gram copy needs unsharded solvers");
    if (!src->have_gram) return fail(CONCORD_ERR_ARG, "source has no Gram matrix");
    DeviceGuard g(dst->dev);
    CK(cudaStreamSynchronize(src->stream));
    int rc = ensure_stage(dst);
    if (rc) return rc;
    CK(launch_unpack_slabs(src->T, dst->stage, src->p, src->w, src->ss, src->ld, src->nblk_launch, src->blk0,
                           dst->stream));
    rc = set_gram_rowmajor(dst, dst->stage, CONCORD_DEVICE);
    if (rc) return rc;
    dst->n = src->n;
    return CONCORD_OK;
}

int concord_solver_take_state(concord_solver* dst, concord_solver* src) {
    if (!dst || !src) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (dst == src) {  // continue in place: the next fit resumes from this solver's own state
        dst->resume = true;
        return CONCORD_OK;
    }
    if (dst->p != src->p || dst->dev != src->dev)
        return fail(CONCORD_ERR_ARG, "solvers differ in p or device (%d/%d vs %d/%d)", dst->p, dst->dev, src->p,
                    src->dev);
    if (dst->G > 1 || dst->rank >= 0 || src->G > 1 || src->rank >= 0)
        return fail(CONCORD_ERR_ARG, "state hand-over needs unsharded solvers");
    if (!dst->have_gram || !src->have_gram || dst->n != src->n) return fail(CONCORD_ERR_ARG, "Gram matrices differ");
    DeviceGuard g(dst->dev);
    CK(cudaStreamSynchronize(src->stream));
    int rc = ensure_stage(dst);
    if (rc) return rc;
    const double* from[2] = {src->Om, src->W};
    double* to[2] = {dst->Om, dst->W};
    const size_t tot = (size_t)dst->nblk_launch * dst->slab;
    for (int k = 0; k < 2; ++k) {  // src slabs -> row-major p x p scratch -> dst slabs, on dst's stream
        CK(cudaMemsetAsync(to[k], 0, sizeof(double) * tot, dst->stream));  // padding as after a cold start
        CK(launch_unpack_slabs(from[k], dst->stage, src->p, src->w, src->ss, src->ld, src->nblk_launch, src->blk0,
                               dst->stream));
        CK(launch_pack_slabs(dst->stage, dst->p, to[k], dst->p, dst->w, dst->ss, dst->ld, dst->nblk_launch, dst->blk0,
                             dst->stream));
    }
    // src is free for other work once this returns (the scheduler hands it to another lane)
    CK(cudaStreamSynchronize(dst->stream));
    dst->resume = true;
    return CONCORD_OK;
}

int concord_solver_layout(concord_solver* s, concord_layout* out) {
    if (!s || !out) return fail(CONCORD_ERR_ARG, "NULL argument");
    out->p = s->p;
    out->slab_width = s->w;
    out->n_shards = s->G;
    out->rank = s->rank;
    out->blocks_per_shard = s->nblk_loc;
    out->blocks_total = s->nblk_tot;
    out->col0 = s->blk0 * s->w < s->p ? s->blk0 * s->w : s->p;
    out->ncols = ncols_local(s);
    out->lag_cap = s->lmax;
    out->kernel = s->qb ? s->qb_D : 0;
    return CONCORD_OK;
}

int concord_solver_destroy(concord_solver* s) {
    if (!s) return CONCORD_OK;
    DeviceGuard g(s->dev);
    if (s->own_stream) cudaStreamSynchronize(s->own_stream);
    cudaFree(s->T);
    cudaFree(s->W);
    cudaFree(s->Om);
    cudaFree(s->tdiag);
    cudaFree(s->stage);
    cudaFree(s->diagd);
    cudaFree(s->Tfull);
    for (int r = 0; r < WFORM_MAX_SHARDS; ++r) {
        if (!s->arena[r]) continue;
        if (s->arena_owned[r]) cudaFree(s->arena[r]);
        else cudaIpcCloseMemHandle(s->arena[r]);
    }
    cudaFree(s->edges);
    if (s->hang) cudaFreeHost(s->hang);
    if (s->yield) cudaFreeHost((void*)s->yield);
    cudaFree(s->status);
    cudaFree(s->rec_delta);
    cudaFree(s->rec_obj);
    cudaFree(s->rec_time);
    cudaFree(s->rec_nnz);
    cudaFree(s->csr_rowptr);
    cudaFree(s->csr_col);
    cudaFree(s->csr_val);
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    delete s;
    return CONCORD_OK;
}

int concord_solver_set_stream(concord_solver* s, void* stream) {
    if (!s) return fail(CONCORD_ERR_ARG, "solver is NULL");
    s->stream = stream ? (cudaStream_t)stream : s->own_stream;
    return CONCORD_OK;
}

void* concord_solver_stream(concord_solver* s) { return s ? (void*)s->stream : nullptr; }

int concord_solver_set_gram(concord_solver* s, const double* T, double n, int32_t where) {
    if (!s || !T) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (!(n >= 1.0)) return fail(CONCORD_ERR_ARG, "n must be at least 1");
    DeviceGuard g(s->dev);
    s->n = n;
    return set_gram_rowmajor(s, T, where);
}

int concord_solver_gram_from_data(concord_solver* s, const double* X, int64_t n, int32_t where) {
    if (!s || !X) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (n < 1) return fail(CONCORD_ERR_ARG, "need at least one observation");
    DeviceGuard g(s->dev);
    const double* Xd = X;
    double* tmp = nullptr;
    if (where == CONCORD_HOST) {
        CK(dalloc(&tmp, (size_t)n * s->p));
        CK(cudaMemcpyAsync(tmp, X, sizeof(double) * (size_t)n * s->p, cudaMemcpyHostToDevice, s->stream));
        Xd = tmp;
    }
    int rc = ensure_stage(s);
    cudaError_t e = rc ? cudaErrorMemoryAllocation : cudaSuccess;
    if (e == cudaSuccess) e = launch_gram_f64(Xd, n, s->p, s->p, s->stage, 0, 0, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (tmp) cudaFree(tmp);
    if (rc) return rc;
    CK(e);
    s->n = (double)n;
    return set_gram_rowmajor(s, s->stage, CONCORD_DEVICE);
}

int concord_solver_gram_from_raw_data(concord_solver* s, const double* X, int64_t n, int32_t where) {
    if (!s || !X) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (n < 1) return fail(CONCORD_ERR_ARG, "need at least one observation");
    DeviceGuard g(s->dev);
    double* tmp = nullptr;
    CK(dalloc(&tmp, (size_t)n * s->p));
    cudaError_t e = cudaMemcpyAsync(tmp, X, sizeof(double) * (size_t)n * s->p,
                                    where == CONCORD_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                    s->stream);
    if (e == cudaSuccess) e = launch_center_columns(tmp, n, s->p, s->p, s->stream);
    int rc = (e == cudaSuccess) ? concord_solver_gram_from_data(s, tmp, n, CONCORD_DEVICE) : CONCORD_OK;
    cudaStreamSynchronize(s->stream);
    cudaFree(tmp);
    CK(e);
    return rc;
}

int concord_solver_get_gram(concord_solver* s, double* T_out, int32_t where) {
    if (!s || !T_out) return fail(CONCORD_ERR_ARG, "NULL argument");
    DeviceGuard g(s->dev);
    return download_slabs(s, s->T, T_out, where);
}

int concord_solver_fit(concord_solver* s, const concord_fit_params* prm, concord_fit_result* res,
                       double* delta_trace, double* objective_trace, double* sweep_seconds) {
    if (!s || !prm) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (!s->have_gram) return fail(CONCORD_ERR_ARG, "no Gram matrix set");
    if (!s->peers_open) return fail(CONCORD_ERR_ARG, "shard peers not opened (concord_shard_open_peers)");
    if (!(prm->lam >= 0.0)) return fail(CONCORD_ERR_ARG, "lam must be nonnegative");
    if (!(prm->delta_tol > 0.0)) return fail(CONCORD_ERR_ARG, "delta_tol must be positive");
    if (prm->max_iter < 1) return fail(CONCORD_ERR_ARG, "max_outer_iterations must be at least 1");
    const int pe = s->p + (s->p & 1);
    if ((long long)prm->max_iter * pe >= (1LL << 31))
        return fail(CONCORD_ERR_ARG, "max_outer_iterations * p too large (%d x %d)", prm->max_iter, pe);
    DeviceGuard g(s->dev);
    int rc = ensure_records(s, prm->max_iter);
    if (rc) return rc;
    const size_t tot = (size_t)s->nblk_launch * s->slab;

    CK(cudaEventRecord(s->ev[0], s->stream));
    if (s->resume) {
        // continue a yielded fit: Omega and W as concord_solver_import_state left them
        s->resume = false;  // consumed (also when rejected below)
        if (prm->omega_init) return fail(CONCORD_ERR_ARG, "omega_init given while an imported state is pending");
    } else if (prm->omega_init) {
        rc = init_warm(s, prm->omega_init, prm->init_where);
        if (rc) return rc;
    } else {
        CK(launch_slab_identity(s->Om, s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->stream));
        CK(cudaMemcpyAsync(s->W, s->T, sizeof(double) * tot, cudaMemcpyDeviceToDevice, s->stream));
    }
    CK(cudaMemsetAsync(s->rec_nnz, 0, sizeof(long long) * prm->max_iter, s->stream));
    CK(cudaEventRecord(s->ev[1], s->stream));

    WformArgs a;
    memset(&a, 0, sizeof(a));
    a.p = s->p;
    a.m = pe - 1;
    a.half = pe / 2;
    a.w = s->w;
    a.slab = s->slab;
    a.W = s->W;
    a.T = s->T;
    a.Om = s->Om;
    a.tdiag = s->tdiag;
    a.diagd = s->diagd;
    a.x = copies(s);
    a.G = s->G;
    a.nblk_loc = s->nblk_loc;
    a.nblk_tot = s->nblk_tot;
    a.blk0 = s->blk0;
    a.sys_scope = (s->rank >= 0 && s->G > 1) ? 1 : 0;
    // testing: the system-scope (NVLink peer) fences and reductions on virtual shards of one device
    if (const char* e = getenv("CONCORD_FORCE_SYS_SCOPE")) a.sys_scope = atoi(e) ? 1 : a.sys_scope;
    a.bar_base = s->bar_base;
    a.it_base = s->it_base;
    a.n = s->n;
    a.shrink = s->n * prm->lam;
    a.delta_tol = prm->delta_tol;
    a.max_iter = prm->max_iter;
    a.want_trace = prm->want_trace ? 1 : 0;
    CK(cudaHostGetDevicePointer((void**)&a.hang, s->hang, 0));
    a.lmax = s->lmax;
    a.rd = s->rd;
    a.rl = s->rl;
    a.rec_delta = s->rec_delta;
    a.rec_obj = s->rec_obj;
    a.rec_time = s->rec_time;
    a.rec_nnz = s->rec_nnz;
    a.share = s->share;
    a.nsh = s->nsh;
    a.stage_ahead = 3;
    if (const char* e = getenv("CONCORD_STAGE_AHEAD")) a.stage_ahead = atoi(e);
    if (a.stage_ahead < 2) a.stage_ahead = 2;
    if (a.stage_ahead > 3) a.stage_ahead = 3;
    a.tdiag_smem = wform_tdiag_in_smem(s->p);
    a.status = s->status;
    unsigned long long* prof = nullptr;
    const bool want_prof = getenv("CONCORD_PHASE_PROFILE") != nullptr;
    if (want_prof) {
        CK(dalloc(&prof, 16));
        CK(cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), s->stream));
    }
    a.prof = prof;
    if (s->qb) {
        QbArgs q;
        memset(&q, 0, sizeof(q));
        q.p = a.p;
        q.m = a.m;
        q.half = a.half;
        q.w = a.w;
        q.slab = s->ss;
        q.ld = (int)s->ld;
        q.slabT = s->Tfull ? s->ssT : s->ss;
        q.ldT = (int)(s->Tfull ? s->ldT : s->ld);
        q.W = a.W;
        q.T = a.T;
        q.Tfull = s->Tfull ? s->Tfull : a.T;
        q.Om = a.Om;
        q.tdiag = a.tdiag;
        q.tdiag_smem = s->qb_td;
        q.nbuf = s->qb_nbuf;
        q.colour_warps_min = 1;
        q.chain_warps = s->qb_cw;
        if (const char* e = getenv("CONCORD_QB_CW")) q.colour_warps_min = atoi(e);
        q.ring_stages = s->qb_ring;
        for (int r = 0; r < s->G; ++r) {
            char* base = static_cast<char*>(s->arena[r]);
            q.x.diagv[r] = reinterpret_cast<double2*>(base + s->L.qb_diagv);
            q.x.stW[r] = reinterpret_cast<double*>(base + s->L.qb_stW);
            q.x.stO[r] = reinterpret_cast<double*>(base + s->L.qb_stO);
            q.x.stT[r] = reinterpret_cast<double*>(base + s->L.qb_stT);
            q.x.dring[r] = reinterpret_cast<double*>(base + s->L.qb_dring);
            q.x.list_rs[r] = reinterpret_cast<int2*>(base + s->L.qb_lrs);
            q.x.list_dn[r] = reinterpret_cast<double2*>(base + s->L.qb_ldn);
            q.x.list_cnt[r] = reinterpret_cast<int*>(base + s->L.qb_lcnt);
            q.x.bar[r] = a.x.bar[r];
            q.x.dmax[r] = a.x.dmax[r];
        }
        q.G = s->G;
        q.nblk_loc = s->nblk_loc;
        q.nblk_tot = s->nblk_tot;
        q.blk0 = s->blk0;
        q.sys_scope = a.sys_scope;
        q.sr = s->qb_sr;
        q.rd = s->qb_rd;
        q.rl = s->qb_rl;
        q.share = s->share;
        q.bar_base = a.bar_base;
        q.it_base = a.it_base;
        q.n = a.n;
        q.shrink = a.shrink;
        q.delta_tol = a.delta_tol;
        q.max_iter = a.max_iter;
        q.want_trace = a.want_trace;
        q.D = s->qb_D;
        q.NB = s->qb_NB;
        {
            // Granlund-Montgomery: l = ceil(log2 d), magic = floor(2^32 (2^l - d) / d) + 1,
            // q = (t + ((b - t) >> 1)) >> (l - 1) with t = umulhi(b, magic), exact for all 32-bit b
            auto magic = [](unsigned d, unsigned& mg, int& sh) {
                int l = 0;
                while ((1ull << l) < d) ++l;
                sh = (d <= 1) ? -1 : l - 1;
                mg = (d <= 1) ? 0u : (unsigned)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
            };
            magic((unsigned)s->qb_NB, q.nb_magic, q.nb_shift);
            magic((unsigned)s->w, q.w_magic, q.w_shift);
            magic((unsigned)(s->w / 2), q.w2_magic, q.w2_shift);
            magic((unsigned)s->nblk_tot, q.nblk_magic, q.nblk_shift);
        }
        q.cellcap = qblock_cellcap(s->share, s->qb_D);
        q.rmax = qblock_rmax(s->share, s->qb_D);
        q.stage_window = 4 * s->qb_D;
        q.rec_delta = a.rec_delta;
        q.rec_obj = a.rec_obj;
        q.rec_time = a.rec_time;
        q.rec_nnz = a.rec_nnz;
        q.status = a.status;
        q.prof = a.prof;
        q.hang = a.hang;
        q.yield = nullptr;
        if (s->G == 1) CK(cudaHostGetDevicePointer((void**)&q.yield, (void*)s->yield, 0));
        CK(launch_pcd_qblock(q, s->nblk_launch, s->stream));
    } else {
        CK(launch_pcd_wform(a, s->nblk_launch, s->stream));
    }
    CK(cudaEventRecord(s->ev[2], s->stream));
    CK(launch_slab_edge_count(s->Om, s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->edges, s->stream));

    int status[2] = {0, 0};
    unsigned long long edges = 0;
    {
        cudaError_t e = cudaMemcpyAsync(status, s->status, sizeof(status), cudaMemcpyDeviceToHost, s->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&edges, s->edges, sizeof(edges), cudaMemcpyDeviceToHost, s->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess && s->hang && s->hang[0] != 0) {
            const long long* h = s->hang;
            static const char* what[3] = {"grid barrier (value, target)", "chain waiting for its stager (block, staged)",
                                          "apply warps idle (phase, epoch, staged, stop)"};
            const int k = (int)(h[0] - 1) < 3 ? (int)(h[0] - 1) : 2;
            return fail(CONCORD_ERR_CUDA,
                        "fit kernel watchdog (no progress for 20 s): CTA %lld at block/phase %lld, %s = %lld %lld %lld %lld; "
                        "CUDA: %s",
                        h[1], h[2], what[k], h[3], h[4], h[5], h[6], cudaGetErrorString(e));
        }
        CK(e);
    }
    const int iters = status[0];
    s->last_iters = iters;
    // every shard ran the same phases: the barrier saw (phases) * nblk_tot arrivals, one per CTA
    // per phase plus the initial publish, minus the final diagonal step's (no arrival after it)
    const unsigned long long phases = (unsigned long long)iters * (unsigned long long)pe;
    if (s->qb)  // one arrival per CTA at the start, then one per block up to the deciding block
        s->bar_base += ((unsigned long long)iters * (unsigned long long)s->qb_NB + 1ull) * (unsigned long long)s->nblk_tot;
    else
        s->bar_base += phases * (unsigned long long)s->nblk_tot;
    s->it_base += iters;
    std::vector<double> dl(iters > 0 ? iters : 1);
    std::vector<unsigned long long> tm(iters + 1);
    // on the solver's stream: a legacy-stream copy could wait for another solver's running fit
    CK(cudaMemcpyAsync(dl.data(), s->rec_delta, sizeof(double) * iters, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(tm.data(), s->rec_time, sizeof(unsigned long long) * (iters + 1), cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (delta_trace)
        for (int i = 0; i < iters; ++i) delta_trace[i] = dl[i];
    if (sweep_seconds)
        for (int i = 0; i < iters; ++i) sweep_seconds[i] = (double)(tm[i + 1] - tm[i]) * 1e-9;
    if (objective_trace) {
        if (prm->want_trace) {
            std::vector<double> ro((size_t)iters * s->nblk_launch * 3);
            CK(cudaMemcpyAsync(ro.data(), s->rec_obj, sizeof(double) * ro.size(), cudaMemcpyDeviceToHost, s->stream));
            CK(cudaStreamSynchronize(s->stream));
            for (int i = 0; i < iters; ++i) {
                double q = 0.0, pen = 0.0, lg = 0.0;
                for (int b = 0; b < s->nblk_launch; ++b) {
                    const double* r = &ro[((size_t)i * s->nblk_launch + b) * 3];
                    q += r[0];
                    pen += r[1];
                    lg += r[2];
                }
                objective_trace[i] = -s->n * lg + 0.5 * q + s->n * prm->lam * pen;
            }
        } else {
            for (int i = 0; i < iters; ++i) objective_trace[i] = NAN;
        }
    }
    if (want_prof) {
        unsigned long long pc[16];
        CK(cudaMemcpy(pc, prof, sizeof(pc), cudaMemcpyDeviceToHost));
        cudaFree(prof);
        int clk_khz = 0;
        cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, s->dev);
        const double ph = (double)pc[3];
        fprintf(stderr, "[concord phase profile] p=%d iters=%d phases=%.0f lmax=%d shards=%d clk=%d kHz (CTA 0)\n",
                s->p, iters, ph, s->lmax, s->G, clk_khz);
        const char* names[15] = {"chain: barrier wait", "chain: stage wait", "chain: publish+share+arrive", "-",
                                 "apply: busy", "apply: idle", "apply: batches", "chain:  publish (tc0)",
                                 "chain:  bar+fence+arrive", "chain:  share (last thread)", "apply:  heads+stage",
                                 "apply:  diagonal steps", "apply:   broadcast bars", "apply:   heads loop (ta0)",
                                 "apply:   stage loop (ta0)"};
        const char* qnames[15] = {"chain: barrier wait", "chain: cells part B", "chain: colours+diag", "-",
                                  "apply: busy", "apply: idle", "apply: batches", "chain:  cells part A (prefetch group)",
                                  "apply:  heads+stage (batches)", "chain:  wait for own stager",
                                  "apply:  stage", "apply:  diagonal steps", "chain:  colour corrections (q0)",
                                  "chain:  colour closed form (q0)", "chain:  colour publish (q0)"};
        if (s->qb) {
            fprintf(stderr, "  (blocked kernel: per-block figures; %d colours per block)\n", s->qb_D);
            for (int i = 0; i < 15; ++i) names[i] = qnames[i];
        }
        for (int i = 0; i < 15; ++i) {
            if (i == 3 || i == 6 || names[i][0] == '-') continue;
            const double us = pc[i] / (clk_khz * 1e-3);
            fprintf(stderr, "  %-30s %12.1f us total  %9.3f us/phase\n", names[i], us, us / (ph > 0 ? ph : 1));
        }
        fprintf(stderr, "  %-30s %12llu (%.2f phases/batch)\n", names[6], pc[6], pc[6] ? ph / pc[6] : 0.0);
        if (s->qb)
            fprintf(stderr, "  %-30s %12.1f us total  %9.3f us/phase\n", "apply:  rows (batches)", pc[15] / (clk_khz * 1e-3),
                    pc[15] / (clk_khz * 1e-3) / (ph > 0 ? ph : 1));
    }
    float setup_ms = 0.f, kernel_ms = 0.f;
    CK(cudaEventElapsedTime(&setup_ms, s->ev[0], s->ev[1]));
    CK(cudaEventElapsedTime(&kernel_ms, s->ev[1], s->ev[2]));
    if (res) {
        res->iterations = iters;
        res->converged = status[1] == 1 ? 1 : 0;
        res->final_delta = iters > 0 ? dl[iters - 1] : INFINITY;
        res->edge_count = (int64_t)edges;
        res->kernel_ms = kernel_ms;
        res->setup_ms = setup_ms;
        res->n_blocks = s->nblk_tot;
        res->slab_width = s->w;
    }
    if (status[1] == 2) return CONCORD_YIELDED;
    if (!status[1]) {
        fail(CONCORD_NOT_CONVERGED, "no convergence after %d outer iterations, final delta %.3e", iters,
             iters > 0 ? dl[iters - 1] : INFINITY);
        return CONCORD_NOT_CONVERGED;
    }
    return CONCORD_OK;
}

int concord_solver_objective_parts(concord_solver* s, double* parts, int32_t cap) {
    if (!s || !parts) return fail(CONCORD_ERR_ARG, "NULL argument");
    DeviceGuard g(s->dev);
    const int k = s->last_iters < cap ? s->last_iters : cap;
    std::vector<double> ro((size_t)k * s->nblk_launch * 3);
    if (k > 0) {
        CK(cudaMemcpyAsync(ro.data(), s->rec_obj, sizeof(double) * ro.size(), cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    }
    for (int i = 0; i < k; ++i) {
        double q = 0.0, pen = 0.0, lg = 0.0;
        for (int b = 0; b < s->nblk_launch; ++b) {
            const double* r = &ro[((size_t)i * s->nblk_launch + b) * 3];
            q += r[0];
            pen += r[1];
            lg += r[2];
        }
        parts[3 * i] = q;
        parts[3 * i + 1] = pen;
        parts[3 * i + 2] = lg;
    }
    return CONCORD_OK;
}

int concord_solver_get_omega(concord_solver* s, double* omega_out, int32_t where) {
    if (!s || !omega_out) return fail(CONCORD_ERR_ARG, "NULL argument");
    DeviceGuard g(s->dev);
    return download_slabs(s, s->Om, omega_out, where);
}

int concord_solver_edge_count(concord_solver* s, int64_t* out) {
    if (!s || !out) return fail(CONCORD_ERR_ARG, "NULL argument");
    DeviceGuard g(s->dev);
    unsigned long long edges = 0;
    CK(launch_slab_edge_count(s->Om, s->p, s->w, s->ss, s->ld, s->nblk_launch, s->blk0, s->edges, s->stream));
    CK(cudaMemcpyAsync(&edges, s->edges, sizeof(edges), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *out = (int64_t)edges;
    return CONCORD_OK;
}

int concord_solver_sweep_stats(concord_solver* s, int64_t* nnz_pairs, int32_t cap, int32_t* count) {
    if (!s || !count) return fail(CONCORD_ERR_ARG, "NULL argument");
    DeviceGuard g(s->dev);
    const int k = s->last_iters < cap ? s->last_iters : cap;
    if (k > 0 && nnz_pairs) {
        CK(cudaMemcpyAsync(nnz_pairs, s->rec_nnz, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    }
    *count = s->last_iters;
    return CONCORD_OK;
}

int concord_solver_check_optimality(concord_solver* s, double lam, double* worst, int64_t* row, int64_t* col) {
    if (!s || !worst || !row || !col) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (s->rank >= 0 && s->G > 1) return fail(CONCORD_ERR_ARG, "check_optimality needs every column on this device");
    if (!s->have_gram || s->last_iters < 1) return fail(CONCORD_ERR_ARG, "no fitted estimate");
    DeviceGuard g(s->dev);
    const int nb = 148 * 4;
    double* bv = nullptr;
    long long* bi = nullptr;
    CK(dalloc(&bv, nb));
    cudaError_t e = dalloc(&bi, nb);
    std::vector<double> hv(nb);
    std::vector<long long> hi(nb);
    if (e == cudaSuccess) e = launch_optimality(s->W, s->Om, s->p, s->w, s->ss, s->ld, s->n, s->n * lam, bv, bi, nb, s->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hv.data(), bv, sizeof(double) * nb, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hi.data(), bi, sizeof(long long) * nb, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    cudaFree(bv);
    cudaFree(bi);
    CK(e);
    double best = -1.0;
    long long bidx = 0;
    for (int k = 0; k < nb; ++k)
        if (hv[k] > best || (hv[k] == best && hi[k] < bidx)) {
            best = hv[k];
            bidx = hi[k];
        }
    *worst = best;
    *row = bidx / s->p;
    *col = bidx % s->p;
    return CONCORD_OK;
}

int concord_solver_estimate_entries(concord_solver* s, int64_t* count, int32_t* ii, int32_t* jj, double* vv,
                                    int64_t cap) {
    if (!s || !count) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (s->rank >= 0 && s->G > 1) return fail(CONCORD_ERR_ARG, "estimate_entries needs every column on this device");
    DeviceGuard g(s->dev);
    const int p = s->p;
    int* rowcnt = nullptr;
    CK(dalloc(&rowcnt, p));
    std::vector<int> hc(p);
    cudaError_t e = launch_triplet_count(s->Om, p, s->w, s->ss, s->ld, rowcnt, s->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), rowcnt, sizeof(int) * p, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    cudaFree(rowcnt);
    CK(e);
    std::vector<long long> off(p + 1, 0);
    for (int i = 0; i < p; ++i) off[i + 1] = off[i] + hc[i];
    *count = off[p];
    if (!ii || !jj || !vv) return CONCORD_OK;  // size query
    if (cap < off[p]) return fail(CONCORD_ERR_ARG, "capacity %lld < %lld entries", (long long)cap, off[p]);
    long long* doff = nullptr;
    int *di = nullptr, *dj = nullptr;
    double* dv = nullptr;
    e = dalloc(&doff, p + 1);
    if (e == cudaSuccess) e = dalloc(&di, off[p]);
    if (e == cudaSuccess) e = dalloc(&dj, off[p]);
    if (e == cudaSuccess) e = dalloc(&dv, off[p]);
    if (e == cudaSuccess) e = cudaMemcpyAsync(doff, off.data(), sizeof(long long) * (p + 1), cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = launch_triplet_write(s->Om, p, s->w, s->ss, s->ld, doff, di, dj, dv, s->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ii, di, sizeof(int) * off[p], cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(jj, dj, sizeof(int) * off[p], cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(vv, dv, sizeof(double) * off[p], cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    cudaFree(doff);
    cudaFree(di);
    cudaFree(dj);
    cudaFree(dv);
    CK(e);
    return CONCORD_OK;
}

}  // extern "C"

namespace {

// Banded Cholesky of the AR(2) truth (unit diagonal, bands 0.45 / 0.40; datagen.py:64-78):
// lb[k*p + i] = L[i+k, i].
int ar2_factor(int p, std::vector<double>& lb) {
    lb.assign(3 * (size_t)p, 0.0);
    for (int i = 0; i < p; ++i) {
        const double a1 = (i >= 1) ? lb[p + (i - 1)] : 0.0;      // L[i, i-1]
        const double a2 = (i >= 2) ? lb[2 * p + (i - 2)] : 0.0;  // L[i, i-2]
        const double d = 1.0 - a1 * a1 - a2 * a2;
        if (!(d > 0.0)) return fail(CONCORD_ERR_ARG, "AR(2) truth is not positive definite at %d", i);
        const double lii = sqrt(d);
        lb[i] = lii;
        if (i + 1 < p) {
            const double l_i1_im1 = (i >= 1) ? lb[2 * p + (i - 1)] : 0.0;  // L[i+1, i-1]
            lb[p + i] = (0.45 - l_i1_im1 * a1) / lii;
        }
        if (i + 2 < p) lb[2 * p + i] = 0.40 / lii;
    }
    return CONCORD_OK;
}

// Centred AR(2) samples on the device: X_dev (n x p). Scratch is allocated here.
int ar2_sample_device(int p, long long n, unsigned long long seed, double* X_dev, cudaStream_t st) {
    std::vector<double> lb;
    int rc = ar2_factor(p, lb);
    if (rc) return rc;
    double *dlb = nullptr, *XT = nullptr, *mean = nullptr;
    cudaError_t e = dalloc(&dlb, lb.size());
    if (e == cudaSuccess) e = dalloc(&XT, (size_t)n * p);
    if (e == cudaSuccess) e = dalloc(&mean, p);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dlb, lb.data(), sizeof(double) * lb.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_ar2_sample(dlb, p, n, seed, XT, mean, X_dev, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dlb);
    cudaFree(XT);
    cudaFree(mean);
    CK(e);
    return CONCORD_OK;
}

// Tree-structured truth (scale-free): parent/lpar/ldiag host arrays of p entries (synth.tree_cholesky).
int tree_sample_device(int p, long long n, unsigned long long seed, const int32_t* parent, const double* lpar,
                       const double* ldiag, double* X_dev, cudaStream_t st) {
    for (int v = 0; v < p; ++v) {
        if (parent[v] >= v || (v > 0 && parent[v] < 0) || (v == 0 && parent[v] != -1))
            return fail(CONCORD_ERR_ARG, "parent[%d] = %d: need parent[0] = -1 and 0 <= parent[v] < v", v, parent[v]);
        if (!(ldiag[v] > 0.0)) return fail(CONCORD_ERR_ARG, "ldiag[%d] must be positive", v);
    }
    int* dpar = nullptr;
    double *dl = nullptr, *XT = nullptr, *mean = nullptr;
    cudaError_t e = cudaMalloc(&dpar, sizeof(int) * (size_t)p);
    if (e == cudaSuccess) e = dalloc(&dl, 2 * (size_t)p);
    if (e == cudaSuccess) e = dalloc(&XT, (size_t)n * p);
    if (e == cudaSuccess) e = dalloc(&mean, p);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dpar, parent, sizeof(int) * (size_t)p, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dl, lpar, sizeof(double) * (size_t)p, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dl + p, ldiag, sizeof(double) * (size_t)p, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_tree_sample(dpar, dl, dl + p, p, n, seed, XT, mean, X_dev, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dpar);
    cudaFree(dl);
    cudaFree(XT);
    cudaFree(mean);
    CK(e);
    return CONCORD_OK;
}

}  // namespace

extern "C" {

int concord_tree_data_f64(int64_t p, int64_t n, uint64_t seed, const int32_t* parent, const double* lpar,
                          const double* ldiag, double* X_out, int32_t where, int32_t device) {
    if (!X_out || !parent || !lpar || !ldiag || p < 2 || p > (1LL << 30) || n < 1)
        return fail(CONCORD_ERR_ARG, "need p >= 2, n >= 1 and non-NULL buffers");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    double* Xd = X_out;
    if (where == CONCORD_HOST) CK(dalloc(&Xd, (size_t)n * p));
    rc = tree_sample_device((int)p, n, seed, parent, lpar, ldiag, Xd, nullptr);
    if (!rc && where == CONCORD_HOST) {
        cudaError_t e = cudaMemcpy(X_out, Xd, sizeof(double) * (size_t)n * p, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = fail(CONCORD_ERR_CUDA, "copy: %s", cudaGetErrorString(e));
    }
    if (where == CONCORD_HOST) cudaFree(Xd);
    return rc;
}

int concord_solver_gram_from_tree(concord_solver* s, int64_t n, uint64_t seed, const int32_t* parent,
                                  const double* lpar, const double* ldiag) {
    if (!s || n < 1 || !parent || !lpar || !ldiag) return fail(CONCORD_ERR_ARG, "bad arguments");
    DeviceGuard g(s->dev);
    double* X = nullptr;
    CK(dalloc(&X, (size_t)n * s->p));
    int rc = tree_sample_device(s->p, n, seed, parent, lpar, ldiag, X, s->stream);
    if (!rc) rc = concord_solver_gram_from_data(s, X, n, CONCORD_DEVICE);
    cudaFree(X);
    return rc;
}

int concord_ar2_data_f64(int64_t p, int64_t n, uint64_t seed, double* X_out, int32_t where, int32_t device) {
    if (!X_out || p < 3 || n < 1) return fail(CONCORD_ERR_ARG, "need p >= 3, n >= 1 and an output buffer");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    double* Xd = X_out;
    if (where == CONCORD_HOST) CK(dalloc(&Xd, (size_t)n * p));
    rc = ar2_sample_device((int)p, n, seed, Xd, nullptr);
    if (!rc && where == CONCORD_HOST) {
        cudaError_t e = cudaMemcpy(X_out, Xd, sizeof(double) * (size_t)n * p, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = fail(CONCORD_ERR_CUDA, "copy: %s", cudaGetErrorString(e));
    }
    if (where == CONCORD_HOST) cudaFree(Xd);
    return rc;
}

int concord_solver_gram_from_ar2(concord_solver* s, int64_t n, uint64_t seed) {
    if (!s || n < 1 || s->p < 3) return fail(CONCORD_ERR_ARG, "bad arguments");
    DeviceGuard g(s->dev);
    double* X = nullptr;
    CK(dalloc(&X, (size_t)n * s->p));
    int rc = ar2_sample_device(s->p, n, seed, X, s->stream);
    if (!rc) rc = concord_solver_gram_from_data(s, X, n, CONCORD_DEVICE);
    cudaFree(X);
    return rc;
}

int concord_device_sm_count(int32_t device, int32_t* out) {
    if (!out) return fail(CONCORD_ERR_ARG, "out is NULL");
    *out = 0;
    int n = 0;
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    *out = n;
    return CONCORD_OK;
}

int concord_blocked_plan(int64_t p, int32_t n_sms, concord_blocked_plan_t* out) {
    if (!out) return fail(CONCORD_ERR_ARG, "out is NULL");
    memset(out, 0, sizeof(*out));
    if (p < 2 || p > (1LL << 30) || n_sms < 1) return fail(CONCORD_ERR_ARG, "bad p or n_sms");
    const int ip = (int)p;
    int w = (ip + n_sms - 1) / n_sms;  // create_common's default single-device slabs, one CTA per SM
    if (w < 8) w = 8;
    w = (w + 1) & ~1;
    {
        const int w4 = (w + 3) & ~3;  // create_common's sector alignment
        if (w4 != w && 10 * ((ip + w4 - 1) / w4) >= 9 * ((ip + w - 1) / w)) w = w4;
    }
    const int nblk = (ip + w - 1) / w;
    const int half = (ip + (ip & 1)) / 2;
    int share = (half + nblk - 1) / nblk;
    if (share < WFORM_SHARE_MIN) share = WFORM_SHARE_MIN < half ? WFORM_SHARE_MIN : half;
    out->slab_width = w;
    out->ctas = nblk;
    out->share = share;
    QbPlan plan;
    if (ip >= 256 && QB_DEFAULT && qblock_plan(ip, nblk, share, QB_DEFAULT_D, true, QB_CHAIN_WARPS, &plan)) {
        out->colours_per_barrier = plan.D;
        out->cell_buffers = plan.nbuf;
        out->tdiag_in_smem = plan.td;
        out->ring_stages = plan.ring;
        out->smem_bytes = (int64_t)plan.smem;
    }
    return CONCORD_OK;
}

int concord_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return fail(CONCORD_ERR_ARG, "bad arguments");
    *out = nullptr;
    CK(cudaHostAlloc(out, bytes > 0 ? (size_t)bytes : 1, cudaHostAllocPortable));
    return CONCORD_OK;
}

int concord_host_free(void* ptr) {
    if (ptr) CK(cudaFreeHost(ptr));
    return CONCORD_OK;
}

int concord_gram_f64(const double* X, int64_t n, int64_t p, double* T_out, int32_t device) {
    if (!X || !T_out) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (n < 1) return fail(CONCORD_ERR_ARG, "need at least one observation");
    if (p < 2) return fail(CONCORD_ERR_ARG, "need at least two variables");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    double *Xd = nullptr, *Td = nullptr;
    CK(dalloc(&Xd, (size_t)n * p));
    cudaError_t e = dalloc(&Td, (size_t)p * p);
    if (e == cudaSuccess) e = cudaMemcpy(Xd, X, sizeof(double) * (size_t)n * p, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_gram_f64(Xd, n, (int)p, p, Td, 0, 0, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(T_out, Td, sizeof(double) * (size_t)p * p, cudaMemcpyDeviceToHost);
    cudaFree(Xd);
    cudaFree(Td);
    CK(e);
    return CONCORD_OK;
}

int concord_center_columns_f64(double* X, int64_t n, int64_t p, int32_t where, int32_t device) {
    if (!X) return fail(CONCORD_ERR_ARG, "NULL argument");
    if (n < 1) return fail(CONCORD_ERR_ARG, "need at least one observation");
    if (p < 1 || p > (1LL << 30)) return fail(CONCORD_ERR_ARG, "bad p");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    double* Xd = X;
    if (where == CONCORD_HOST) {
        CK(dalloc(&Xd, (size_t)n * p));
        cudaError_t e = cudaMemcpy(Xd, X, sizeof(double) * (size_t)n * p, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(Xd);
            CK(e);
        }
    }
    cudaError_t e = launch_center_columns(Xd, n, (int)p, p, nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (where == CONCORD_HOST) {
        if (e == cudaSuccess) e = cudaMemcpy(X, Xd, sizeof(double) * (size_t)n * p, cudaMemcpyDeviceToHost);
        cudaFree(Xd);
    }
    CK(e);
    return CONCORD_OK;
}

int concord_pcd_fit(const double* T, int64_t p, double n, const concord_fit_params* prm, double* omega_out,
                    concord_fit_result* res, double* delta_trace, double* objective_trace,
                    double* sweep_seconds, int32_t device) {
    concord_solver* s = nullptr;
    int rc = concord_solver_create(p, device, 0, &s);
    if (rc) return rc;
    rc = concord_solver_set_gram(s, T, n, CONCORD_HOST);
    int fit_rc = rc;
    if (!rc) fit_rc = concord_solver_fit(s, prm, res, delta_trace, objective_trace, sweep_seconds);
    if ((fit_rc == CONCORD_OK || fit_rc == CONCORD_NOT_CONVERGED) && omega_out) {
        std::string keep = g_err;
        rc = concord_solver_get_omega(s, omega_out, CONCORD_HOST);
        if (rc == CONCORD_OK) g_err = keep;
        else fit_rc = rc;
    }
    concord_solver_destroy(s);
    return fit_rc;
}

// ------------------------------------------------------------ exact protocol
namespace {
struct ExactBufs {
    double* om = nullptr;
    double* t = nullptr;
    long long* rs = nullptr;
    long long* ss = nullptr;
    long long* off = nullptr;
    unsigned long long* bar = nullptr;
    ~ExactBufs() {
        cudaFree(om);
        cudaFree(t);
        cudaFree(rs);
        cudaFree(ss);
        cudaFree(off);
        cudaFree(bar);
    }
};

int exact_common(ExactBufs& b, double* om, const double* t, int64_t p) {
    const size_t bytes = sizeof(double) * (size_t)p * p;
    CK(dalloc(&b.om, (size_t)p * p));
    CK(dalloc(&b.t, (size_t)p * p));
    CK(cudaMemcpy(b.om, om, bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b.t, t, bytes, cudaMemcpyHostToDevice));
    return CONCORD_OK;
}
}  // namespace

int concord_pcd_sweep_exact(double* om, const double* t, int64_t p, double n, double shrink,
                            const int64_t* rs, const int64_t* ss, const int64_t* offsets, int64_t nrounds,
                            int32_t device) {
    if (!om || !t || !offsets || p < 1 || nrounds < 0) return fail(CONCORD_ERR_ARG, "bad arguments");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    ExactBufs b;
    rc = exact_common(b, om, t, p);
    if (rc) return rc;
    const long long m = offsets[nrounds];
    CK(dalloc(&b.rs, m));
    CK(dalloc(&b.ss, m));
    CK(dalloc(&b.off, nrounds + 1));
    CK(dalloc(&b.bar, 1));
    if (m) {
        CK(cudaMemcpy(b.rs, rs, sizeof(long long) * m, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(b.ss, ss, sizeof(long long) * m, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(b.off, offsets, sizeof(long long) * (nrounds + 1), cudaMemcpyHostToDevice));
    CK(launch_pcd_sweep_exact(b.om, b.t, (int)p, n, shrink, b.rs, b.ss, b.off, (int)nrounds, b.bar, nullptr));
    CK(cudaMemcpy(om, b.om, sizeof(double) * (size_t)p * p, cudaMemcpyDeviceToHost));
    return CONCORD_OK;
}

int concord_u2_sweep_exact(double* om, const double* t, int64_t p, double n, double shrink, const int64_t* rs,
                           const int64_t* ss, int64_t npairs, int32_t device) {
    if (!om || !t || p < 1 || npairs < 0) return fail(CONCORD_ERR_ARG, "bad arguments");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    ExactBufs b;
    rc = exact_common(b, om, t, p);
    if (rc) return rc;
    CK(dalloc(&b.rs, npairs));
    CK(dalloc(&b.ss, npairs));
    if (npairs) {
        CK(cudaMemcpy(b.rs, rs, sizeof(long long) * npairs, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(b.ss, ss, sizeof(long long) * npairs, cudaMemcpyHostToDevice));
    }
    CK(launch_u2_sweep_exact(b.om, b.t, (int)p, n, shrink, b.rs, b.ss, npairs, nullptr));
    CK(cudaMemcpy(om, b.om, sizeof(double) * (size_t)p * p, cudaMemcpyDeviceToHost));
    return CONCORD_OK;
}

int concord_cd_sweep_exact(double* om, const double* t, int64_t p, double n, double shrink, int32_t device) {
    if (!om || !t || p < 1) return fail(CONCORD_ERR_ARG, "bad arguments");
    int rc = check_device(device);
    if (rc) return rc;
    DeviceGuard g(device);
    ExactBufs b;
    rc = exact_common(b, om, t, p);
    if (rc) return rc;
    CK(launch_cd_sweep_exact(b.om, b.t, (int)p, n, shrink, nullptr));
    CK(cudaMemcpy(om, b.om, sizeof(double) * (size_t)p * p, cudaMemcpyDeviceToHost));
    return CONCORD_OK;
}

}  // extern "C"
