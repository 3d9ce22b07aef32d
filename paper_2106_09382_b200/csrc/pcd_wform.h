// Internal C++ interface of the W-form persistent kernel (not the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef WFORM_THREADS
#define WFORM_THREADS 512
#endif
#ifndef WFORM_CHAIN_WARPS
#define WFORM_CHAIN_WARPS 4     // warps 0..3: publish / closed forms / grid barrier (the colour chain)
#endif
#ifndef WFORM_PAIR_CAP
#define WFORM_PAIR_CAP 1024     // delta-list pairs staged in shared memory per apply chunk
#endif
#ifndef WFORM_SHARE_MIN
#define WFORM_SHARE_MIN 1       // closed forms per share CTA per colour (fewer, longer delta-list segments)
#endif
#ifndef WFORM_BATCH
#define WFORM_BATCH 8           // colour phases one apply batch may cover
#endif
#ifndef WFORM_STAGE_SLOTS
#define WFORM_STAGE_SLOTS 5     // publish stages in flight (shared memory ring)
#endif
#ifndef WFORM_MAX_LAG
#define WFORM_MAX_LAG 8         // max phases the apply warps may trail the chain
#endif
#define WFORM_MAX_BLOCKS 1024
#define WFORM_MAX_SHARDS 8       // copies of the exchange buffers (GPUs, or virtual shards on one GPU)
#define WFORM_DMAX_RING 4        // per-sweep max |delta| accumulators (ring over sweeps)

namespace concord {

// Exchange buffers.  Every shard holds a full copy; writers store into all
// copies (local HBM, or a peer GPU's HBM over NVLink), readers read their own.
struct WformCopies {
    double2* pub[WFORM_MAX_SHARDS];             // [3][p] published (W[x,c], Om[x,c]) per phase mod 3
    double* dring[WFORM_MAX_SHARDS];            // [rd][p] per-row delta of each recent phase
    int2* list_rs[WFORM_MAX_SHARDS];            // [rl][nblk_tot][share] non-zero pairs of a colour
    double2* list_dn[WFORM_MAX_SHARDS];         // [rl][nblk_tot][share] (delta, new value)
    int* list_cnt[WFORM_MAX_SHARDS];            // [rl][nblk_tot] segment lengths
    unsigned long long* bar[WFORM_MAX_SHARDS];  // grid-barrier arrival counter (all CTAs of all shards)
    unsigned long long* dmax[WFORM_MAX_SHARDS]; // [WFORM_DMAX_RING] per-sweep max |off-diagonal delta| bits
};

struct WformArgs {
    int p;          // problem size
    int m;          // rounds per sweep = p_even - 1 (phase m of a sweep is the diagonal step)
    int half;       // pairs per round = p_even / 2
    int w;          // slab width (columns per CTA), even
    long long slab; // p * w doubles per slab
    double* W;      // slab-major p x (nblk*w): W = Omega * T
    const double* T;
    double* Om;     // slab-major dense Omega
    const double* tdiag;
    double2* diagd; // [launch CTAs][p] (delta, new) of the last diagonal step, per CTA
    WformCopies x;  // exchange buffers, one copy per shard
    int G;          // shards
    int nblk_loc;   // CTAs (column slabs) per shard
    int nblk_tot;   // CTAs over all shards
    int blk0;       // global index of this launch's first CTA (its first slab)
    int sys_scope;  // 1: shards are separate GPUs (system-scope fences for peer stores)
    unsigned long long bar_base;  // arrival count of the barrier at the start of this fit (same on all shards)
    int it_base;                  // sweeps run by earlier fits (indexes the dmax ring)
    double n;       // sample count (GramMatrix.n)
    double shrink;  // n * lam (solver.py:285)
    double delta_tol;
    int max_iter;
    int want_trace;
    int lmax;       // lag cap of the apply warps behind the chain (<= WFORM_MAX_LAG, <= m)
    int rd;         // dring slots (>= lmax + 3)
    int rl;         // delta-list ring slots (>= lmax + 4)
    double* rec_delta;              // [max_iter]
    double* rec_obj;                // [max_iter][nblk][3]: <W,Om> part, sum_{i<j}|om|, sum log om_ii
    unsigned long long* rec_time;   // [max_iter + 1] globaltimer ns
    long long* rec_nnz;             // [max_iter] non-zero off-diagonal deltas per sweep, this launch (zeroed)
    int share;                      // pairs per share CTA per colour
    int nsh;                        // CTAs that evaluate closed forms (ceil(half / share))
    int stage_ahead;                // publishes staged beyond the chain's phase
    int tdiag_smem;                 // 1: the T diagonal is copied into shared memory
    int* status;                    // [0] iterations, [1] converged
    unsigned long long* prof;       // optional [16] cycle counters (CTA 0), or NULL
    long long* hang;  // [8] mapped host memory: watchdog report (what+1, CTA, phase/block, 4 values)
};

// Temporally blocked variant (pcd_qblock.cu): D colour phases per grid barrier.
#ifndef QB_DMAX
#define QB_DMAX 4
#endif
#ifndef QB_DEFAULT
#define QB_DEFAULT 1        // 1: single-device solvers use the temporally blocked kernel by default
#endif
#ifndef QB_CHAIN_WARPS
#define QB_CHAIN_WARPS 6     // chain warps of the blocked kernel (the block's cells are loaded in parallel)
#endif
#define WFORM_CHAIN_WARPS_QB QB_CHAIN_WARPS
#ifndef QB_DEFAULT_D
#define QB_DEFAULT_D 4
#endif
// Exchange buffers of the blocked kernel, one copy per shard (like WformCopies): writers store
// into every copy (local HBM, or a peer GPU's over NVLink), readers read their shard's copy.
struct QbCopies {
    double2* diagv[WFORM_MAX_SHARDS];       // [p] (delta, new) of the latest diagonal step
    double* stW[WFORM_MAX_SHARDS];          // [sr][p] staged cell values (W at the block's stage watermark)
    double* stO[WFORM_MAX_SHARDS];          // [sr][p] staged Omega of the cells
    double* stT[WFORM_MAX_SHARDS];          // [sr][QB_DMAX-1][p] staged T entries of the block's earlier phases
    double* dring[WFORM_MAX_SHARDS];        // [rd][p] per-row delta of each recent phase
    int2* list_rs[WFORM_MAX_SHARDS];        // [rl][nblk_tot][share]
    double2* list_dn[WFORM_MAX_SHARDS];
    int* list_cnt[WFORM_MAX_SHARDS];        // [rl][nblk_tot]
    unsigned long long* bar[WFORM_MAX_SHARDS];   // grid-barrier arrivals (all CTAs of all shards)
    unsigned long long* dmax[WFORM_MAX_SHARDS];  // [WFORM_DMAX_RING]
};
struct QbArgs {
    int p, m, half, w;
    long long slab;        // stride between this launch's slabs (p*w: slab layout; w: row-major layout)
    int ld;                // row stride of W, T, Om (w: slab layout; the launch's columns: row-major)
    long long slabT;       // the same two strides for Tfull
    int ldT;
    double* W;             // this launch's slabs
    const double* T;       // this launch's slabs
    const double* Tfull;   // every slab of T (== T unless a process shard): the cells' T entries
    double* Om;
    const double* tdiag;
    int tdiag_smem;
    QbCopies x;            // exchange buffers, one copy per shard
    int G;                 // shards
    int nblk_loc;          // CTAs per shard
    int nblk_tot;          // CTAs over all shards
    int blk0;              // global index of this launch's first CTA
    int sys_scope;         // 1: shards are separate GPUs (system-scope fences for the peer stores)
    int sr;                // stage slots (phases)
    int rd;
    int rl;
    int share;
    unsigned long long bar_base;
    int it_base;
    double n, shrink, delta_tol;
    int max_iter, want_trace;
    int D, NB;             // phases per block, blocks per sweep
    unsigned nb_magic;     // b / NB as a multiply-shift (host-computed, Granlund-Montgomery)
    int nb_shift;          // -1 when NB == 1
    unsigned w_magic, w2_magic;  // the same for the slab width w and w/2 (row-stream cursors)
    int w_shift, w2_shift;
    unsigned nblk_magic;   // and for the CTA count (segments per phase of the delta lists)
    int nblk_shift;
    int cellcap, rmax;     // shared-memory sizing of the block cells
    int stage_window;      // max phases a stage may be brought forward over
    double* rec_delta;
    double* rec_obj;       // [max_iter][launch CTAs][3]
    unsigned long long* rec_time;
    long long* rec_nnz;    // this launch's pairs (a process shard's part of the sweep)
    int* status;
    unsigned long long* prof;
    long long* hang;       // [8] mapped host memory: watchdog report (what+1, CTA, block, 4 values)
    const volatile int* yield;  // mapped host flag: stop at the next sweep end (resumable); NULL = never
    int nbuf;              // cell buffers: 2 = next block's cells built during the colours
    int ring_stages;       // cp.async row-ring depth (2, 4 or 6)
    int colour_warps_min;  // lower bound on the colour group's warps (tuning)
    int chain_warps;       // kernel variant: 4, 6 or 8 chain warps
};
int qblock_cellcap(int share, int D);
int qblock_rmax(int share, int D);
// Chain-warp variants of the blocked kernel: 6 (default), 4 (apply-heavy), 8 (chain-heavy).
bool qblock_variant_ok(int chain_warps);
size_t qblock_smem_bytes(int chain_warps, int p, int nblk, int share, int D, int tdiag_smem, int nbuf,
                         int ring_stages);
int qblock_colour_warps(int chain_warps, int share, int D);
cudaError_t launch_pcd_qblock(const QbArgs& args, int nblk, cudaStream_t st);
// Raise the variant's dynamic shared-memory limit to smem now (solver creation), so no launch
// has to set the attribute while another fit runs.
cudaError_t qblock_reserve_smem(int chain_warps, size_t smem);
namespace qb4 {
size_t smem_bytes(int p, int nblk, int share, int D, int tdiag_smem, int nbuf, int ring_stages);
int colour_warps_host(int share, int D);
cudaError_t launch(const QbArgs& args, int nblk, cudaStream_t st);
cudaError_t reserve_smem(size_t smem);
}
namespace qb6 {
size_t smem_bytes(int p, int nblk, int share, int D, int tdiag_smem, int nbuf, int ring_stages);
int colour_warps_host(int share, int D);
cudaError_t launch(const QbArgs& args, int nblk, cudaStream_t st);
cudaError_t reserve_smem(size_t smem);
}
namespace qb8 {
size_t smem_bytes(int p, int nblk, int share, int D, int tdiag_smem, int nbuf, int ring_stages);
int colour_warps_host(int share, int D);
cudaError_t launch(const QbArgs& args, int nblk, cudaStream_t st);
cudaError_t reserve_smem(size_t smem);
}

// Lag cap for a slab width (bounded by the stage ring's shared memory) and m.
int wform_lag_cap(int w, int m);
int wform_tdiag_in_smem(int p);
size_t wform_smem_bytes(int w, int p, int nblk, int lmax);

cudaError_t launch_pcd_wform(const WformArgs& args, int nblk, cudaStream_t st);
cudaError_t wform_max_blocks(int w, int p, int nblk_tot, int* max_blocks);
// Slab-layout helpers.  `nblk` slabs of width w starting at global column block
// blk0 (columns [blk0*w, (blk0+nblk)*w) clipped to p).
cudaError_t launch_pack_slabs(const double* src, long long ld, double* dst, int p, int w, long long ss, long long rs,
                              int nblk, int blk0, cudaStream_t st);
// Slabs -> row-major p x ncols block (ld = ncols) of the columns the slabs hold.
cudaError_t launch_unpack_slabs(const double* src, double* dst, int p, int w, long long ss, long long rs, int nblk,
                                int blk0, cudaStream_t st);
cudaError_t launch_slab_identity(double* slab, int p, int w, long long ss, long long rs, int nblk, int blk0,
                                 cudaStream_t st);
cudaError_t launch_slab_edge_count(const double* slab, int p, int w, long long ss, long long rs, int nblk, int blk0,
                                   unsigned long long* out, cudaStream_t st);
cudaError_t launch_wform_init_csr(const long long* rowptr, const int* colidx, const double* vals, const double* Tslab,
                                  double* Wslab, int p, int w, long long ss, long long rs, int nblk, cudaStream_t st);
// Diagonal of a row-major p x p matrix (the replicated T diagonal).
cudaError_t launch_rowmajor_diag(const double* src, double* diag, int p, cudaStream_t st);

// Exact (direct-form) reference-protocol sweeps, pcd_exact.cu.
cudaError_t launch_pcd_sweep_exact(double* om, const double* t, int p, double n, double shrink,
                                   const long long* rs, const long long* ss, const long long* offsets,
                                   int nrounds, unsigned long long* bar, cudaStream_t st);
cudaError_t launch_u2_sweep_exact(double* om, const double* t, int p, double n, double shrink,
                                  const long long* rs, const long long* ss, long long npairs, cudaStream_t st);
cudaError_t launch_cd_sweep_exact(double* om, const double* t, int p, double n, double shrink, cudaStream_t st);

// Diagnostics on the slab-resident estimate, diag.cu.
cudaError_t launch_optimality(const double* W, const double* Om, int p, int w, long long ss, long long rs, double n,
                              double weight,
                              double* blk_val, long long* blk_idx, int nblocks, cudaStream_t st);
cudaError_t launch_triplet_count(const double* Om, int p, int w, long long ss, long long rs, int* rowcnt,
                                 cudaStream_t st);
cudaError_t launch_triplet_write(const double* Om, int p, int w, long long ss, long long rs, const long long* rowoff,
                                 int* ti, int* tj,
                                 double* tv, cudaStream_t st);

// On-device AR(2) samples (datagen.cu): centred X (n x p row-major); XT (p x n) and mean (p) are scratch.
cudaError_t launch_tree_sample(const int* parent, const double* lpar, const double* ldiag, int p, long long n,
                               unsigned long long seed, double* XT, double* mean, double* X, cudaStream_t st);
cudaError_t launch_ar2_sample(const double* lb, int p, long long n, unsigned long long seed, double* XT, double* mean,
                              double* X, cudaStream_t st);

// FP64 DMMA Gram / GEMM, gram.cu.  T = X^T X (X: n x p row-major, leading dim ldx).
// out_mode 0: row-major p x p (ld = p); 1: slab-major with width w.
cudaError_t launch_center_columns(double* X, long long n, int p, long long ldx, cudaStream_t st);
cudaError_t launch_gram_f64(const double* X, long long n, int p, long long ldx, double* out, int out_mode, int w,
                            cudaStream_t st);

}  // namespace concord
