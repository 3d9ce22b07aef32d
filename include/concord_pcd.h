/*
 * concord_pcd.h -- C ABI of the B200-native CONCORD-PCD solver
 * (libconcord_b200.so, built from paper_2106_09382_b200/csrc/).
 *
 * Drop-in boundary for the reference package `parconcord`
 * (/root/reference/pkg/src/parconcord).  Plain pointers and sizes only; no
 * C++ exceptions or torch types cross this boundary.  Every function returns
 * CONCORD_OK (0) or a negative code; concord_last_error() describes the last
 * failure on the calling thread.  Matrices are row-major float64, p x p
 * (n x p for data), exactly as the reference's numpy arrays.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/parconcord):
 *   concord_gram_f64 / concord_solver_gram_from_data  -> model.compute_gram         model.py:190-197
 *   concord_solver_fit / concord_pcd_fit               -> solver.pcd_fit            solver.py:254-294
 *                                                         (sweeps _ckernels.pcd_sweep _ckernels.pyx:68-102,
 *                                                          delta solver.py:287, objective model.py:210-217)
 *   concord_solver_edge_count                          -> model.edge_count          model.py:249-253
 *   concord_pcd_sweep_exact                            -> _ckernels.pcd_sweep       _ckernels.pyx:68-102
 *   concord_u2_sweep_exact                             -> _ckernels.u2_sweep        _ckernels.pyx:105-118
 *   concord_cd_sweep_exact                             -> _ckernels.cd_sweep        _ckernels.pyx:53-65
 */
#ifndef CONCORD_PCD_H
#define CONCORD_PCD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CONCORD_ABI_VERSION 2

/* Return codes. */
#define CONCORD_OK 0
#define CONCORD_YIELDED 1              /* the fit stopped at a sweep end on request; resumable   */
#define CONCORD_ERR_ARG (-1)           /* bad dimension / argument (DimensionError, ValueError) */
#define CONCORD_NOT_CONVERGED (-2)     /* iteration cap hit; outputs are valid (NotConverged)   */
#define CONCORD_ERR_CUDA (-3)          /* CUDA runtime error                                    */
#define CONCORD_ERR_ZERO_VARIANCE (-4) /* t_ii <= 0 (ZeroVarianceColumn)                        */
#define CONCORD_ERR_NO_DEVICE (-5)     /* no CUDA device                                        */
#define CONCORD_ERR_OOM (-6)           /* device allocation failed                              */

/* Where a caller buffer lives. */
#define CONCORD_HOST 0
#define CONCORD_DEVICE 1

typedef struct concord_solver concord_solver;

/* Bytes of one shard's exported exchange-buffer handle (a cudaIpcMemHandle_t). */
#define CONCORD_SHARD_HANDLE_BYTES 64

/* Column partition of a solver (or of one shard of a multi-GPU solver). */
typedef struct {
    int64_t p;
    int32_t slab_width;       /* columns per CTA                                            */
    int32_t n_shards;         /* GPUs (or virtual shards) the columns are split over        */
    int32_t rank;             /* this process's shard, -1 when every shard is local         */
    int32_t blocks_per_shard; /* CTAs (column slabs) per shard                              */
    int32_t blocks_total;
    int64_t col0;             /* first column this solver holds                             */
    int64_t ncols;            /* columns this solver holds (p unless it is one shard)       */
    int32_t lag_cap;          /* phases the apply warps may trail the colour chain          */
    int32_t kernel;           /* 0: per-phase chain (pcd_wform_kernel), D >= 1: temporally   */
                              /*    blocked chain with D colours per barrier (pcd_qblock)    */
} concord_layout;

typedef struct {
    double lam;          /* penalty; the soft threshold is n*lam (solver.py:285)           */
    double delta_tol;    /* stop when max |Omega_new - Omega_old| < delta_tol (solver.py:290) */
    int32_t max_iter;    /* max_outer_iterations                                            */
    int32_t want_trace;  /* 1: fused objective trace per sweep                              */
    const double* omega_init; /* NULL = identity (model.py:158-166), else p x p warm start  */
    int32_t init_where;  /* CONCORD_HOST / CONCORD_DEVICE for omega_init                    */
    int32_t reserved;
} concord_fit_params;

typedef struct {
    int32_t iterations;  /* sweeps run                                                      */
    int32_t converged;   /* 1 if final_delta < delta_tol                                    */
    double final_delta;  /* max |delta| of the last sweep                                   */
    int64_t edge_count;  /* exact non-zeros of the strict upper triangle                    */
    double kernel_ms;    /* CUDA-event time of the persistent sweep kernel                  */
    double setup_ms;     /* CUDA-event time of W/Omega initialisation before the kernel     */
    int32_t n_blocks;    /* CTAs (column slabs) used                                        */
    int32_t slab_width;  /* columns per slab                                                */
} concord_fit_result;

/* ---- library / device ------------------------------------------------- */
int concord_abi_version(void);
const char* concord_last_error(void);
int concord_device_count(int* count);

/* ---- device-resident solver (one per problem size and device) ---------- */
/* n_blocks: 0 = automatic slab count; otherwise the number of column slabs. */
int concord_solver_create(int64_t p, int32_t device, int32_t n_blocks, concord_solver** out);
int concord_solver_destroy(concord_solver* s);
/* The same solver with its columns split over n_shards virtual shards on ONE
 * device: every exchange buffer is replicated n_shards times and written by
 * all shards, exactly as the multi-GPU solver does over NVLink.
 * Results are bitwise identical for every n_shards. */
int concord_solver_create_sharded(int64_t p, int32_t device, int32_t n_blocks, int32_t n_shards,
                                  concord_solver** out);
int concord_solver_layout(concord_solver* s, concord_layout* out);
/* Chain-warp variant of the blocked kernel for this solver's fits: 6 (default), 4 (apply-heavy:
 * dense fits), 8 (chain-heavy: sparse fits on a small share of the SMs).  4 and 8 align the roles
 * to warp groups and redistribute registers between them with setmaxnreg.  Results are bitwise
 * identical for every variant.  No reference counterpart (a scheduling knob). */
int concord_solver_set_chain_warps(concord_solver* s, int32_t chain_warps);

/* ---- multi-GPU: one process per GPU, column-sharded --------- */
/* Shard `rank` of n_shards.  Exchange the handles (all-gather of
 * CONCORD_SHARD_HANDLE_BYTES per rank, rank order) and open the peers before
 * the first fit; every rank then calls concord_solver_fit concurrently.
 * set_gram / gram_from_data take the FULL T / X; get_omega / get_gram return
 * this shard's p x ncols column block (concord_solver_layout). */
int concord_shard_create(int64_t p, int32_t n_shards, int32_t rank, int32_t device, int32_t n_blocks,
                         concord_solver** out);
int concord_shard_ipc_handle(concord_solver* s, void* handle_out);
int concord_shard_open_peers(concord_solver* s, const void* handles);
/* Use a caller stream (cudaStream_t as void*); NULL restores the solver's own. */
int concord_solver_set_stream(concord_solver* s, void* stream);
void* concord_solver_stream(concord_solver* s);
/* GramMatrix (model.py:81-103): T p x p row-major and the sample count n. */
int concord_solver_set_gram(concord_solver* s, const double* T, double n, int32_t where);
/* compute_gram (model.py:190-197) on the device from centred data X (n x p). */
int concord_solver_gram_from_data(concord_solver* s, const double* X, int64_t n, int32_t where);
/* center_columns + compute_gram (model.py:182-197; the CLI's load path, cli.py:101-102) on the
 * device from RAW data X (n x p): the column means are bitwise numpy's x.mean(axis=0). */
int concord_solver_gram_from_raw_data(concord_solver* s, const double* X, int64_t n, int32_t where);
int concord_solver_get_gram(concord_solver* s, double* T_out, int32_t where);
/* pcd_fit (solver.py:254-294).  delta_trace / objective_trace / sweep_seconds
 * may be NULL, else hold max_iter doubles.  Returns CONCORD_NOT_CONVERGED when
 * the cap is hit (results valid, like NotConverged.report), and CONCORD_YIELDED
 * when concord_solver_request_yield stopped it at a sweep end (below). */
int concord_solver_fit(concord_solver* s, const concord_fit_params* prm, concord_fit_result* res,
                       double* delta_trace, double* objective_trace, double* sweep_seconds);
int concord_solver_get_omega(concord_solver* s, double* omega_out, int32_t where);
/* ---- moving a running fit to a solver with more SMs (no reference counterpart: the
 * lambda-path scheduler's lane hand-over, python/paper_2106_09382_b200/solver.py) ---
 * request_yield(on=1): the blocked fit running on this solver (or its next one) stops at the
 * end of its current sweep unless that sweep converged or hit max_iter; concord_solver_fit then
 * returns CONCORD_YIELDED with the sweeps run so far.  Thread-safe (a mapped host flag); the
 * flag stays set until request_yield(s, 0).  Unsharded solvers only.
 * export_state: Omega and the maintained W = Omega T as p x p row-major.
 * import_state: the next fit on this solver continues from (Omega, W) instead of the identity /
 * omega_init; the continuation is bitwise the uninterrupted fit (W is carried, not recomputed),
 * for any pair of slab layouts. */
int concord_solver_request_yield(concord_solver* s, int32_t on);
int concord_solver_export_state(concord_solver* s, double* omega_out, double* w_out, int32_t where);
int concord_solver_import_state(concord_solver* s, const double* omega, const double* w, int32_t where);
/* The two steps above device to device: dst (same p, device and Gram, any slab count) continues
 * src's yielded fit with its next concord_solver_fit.  Enqueued on dst's stream after src's
 * stream drained, and complete on return (src is free for other work); src is unchanged.
 * dst == src: the next fit resumes in place. */
int concord_solver_take_state(concord_solver* dst, concord_solver* src);
/* Allocate now what fits of up to max_iter sweeps and state moves allocate lazily (the p x p
 * scratch, the per-sweep records): a solver that joins a running path must not allocate (or
 * free) device memory on the way, which can wait for the other lanes' kernels. */
int concord_solver_reserve(concord_solver* s, int32_t max_iter);
/* dst's T (and n) := src's, device to device (any two slab layouts, same p and device). */
int concord_solver_copy_gram(concord_solver* dst, concord_solver* src);
/* Per-sweep objective partial sums of this solver's columns for the last fit:
 * parts[3*i .. 3*i+2] = (<W,Omega>, sum_{i<j}|omega_ij|, sum log omega_ii)
 * (a shard's partials add up across shards). */
int concord_solver_objective_parts(concord_solver* s, double* parts, int32_t cap);
int concord_solver_edge_count(concord_solver* s, int64_t* out);
/* check_optimality (model.py:256-289) of the last fit on the device, with
 * M = Omega*T taken from the maintained W: worst stationarity violation and
 * its coordinate (row <= col, 0-based; first in row-major order on ties). */
int concord_solver_check_optimality(concord_solver* s, double lam, double* worst, int64_t* row, int64_t* col);
/* The entries write_estimate (fileio.py:87-95) stores -- every diagonal and
 * every exact non-zero with i < j -- compacted on the device in (i, j)
 * order, 0-based.  NULL ii/jj/vv: only *count is set (size query). */
int concord_solver_estimate_entries(concord_solver* s, int64_t* count, int32_t* ii, int32_t* jj, double* vv,
                                    int64_t cap);
/* Non-zero off-diagonal deltas of each sweep of the last fit (the row streams
 * the kernel applied; used for the roofline's algorithmic bytes).  Copies
 * min(cap, iterations) entries, *count = iterations of the last fit. */
int concord_solver_sweep_stats(concord_solver* s, int64_t* nnz_pairs, int32_t cap, int32_t* count);

/* ---- synthetic data on the device ------------------------- */
/* Centred samples of N(0, inv(ar2_precision(p))) (datagen.py:64-78, 135-154):
 * same distribution as the reference sampler, a counter-based (Philox) random
 * stream, O(p n) work, no host copy of X when the Gram is built in place. */
int concord_ar2_data_f64(int64_t p, int64_t n, uint64_t seed, double* X_out, int32_t where, int32_t device);
int concord_solver_gram_from_ar2(concord_solver* s, int64_t n, uint64_t seed);
/* Scale-free truth (datagen.py:99-132): centred N(0, inv(truth)) samples for a tree-structured
 * truth given by its fill-free Cholesky factor in leaves-first order -- parent[v] < v
 * (parent[0] = -1), L[v,v] = ldiag[v], L[parent[v], v] = lpar[v] (synth.tree_cholesky) --
 * drawn on the device (Philox) in O(p n); the solver variant builds T in place. */
int concord_tree_data_f64(int64_t p, int64_t n, uint64_t seed, const int32_t* parent, const double* lpar,
                          const double* ldiag, double* X_out, int32_t where, int32_t device);
int concord_solver_gram_from_tree(concord_solver* s, int64_t n, uint64_t seed, const int32_t* parent,
                                  const double* lpar, const double* ldiag);

/* ---- pinned host buffers for fast H2D/D2H of T and Omega ---------------- */
/* Kernel plan the library chooses for a p x p problem on one device with n_sms SMs (one CTA per
 * SM, default slab layout): the temporally blocked fit kernel with colours_per_barrier colours
 * per grid barrier and the given shared-memory plan, or colours_per_barrier = 0 for the
 * per-phase kernel.  Host-only (no device needed).  Replaces no reference interface: the
 * reference runs one host loop for every p (solver.py:254-294). */
typedef struct {
    int32_t colours_per_barrier; /* D; 0 = per-phase kernel */
    int32_t cell_buffers;        /* 2 = next block's cells built during the colours */
    int32_t tdiag_in_smem;
    int32_t ring_stages;         /* cp.async row-ring depth */
    int64_t smem_bytes;          /* dynamic shared memory per CTA */
    int32_t slab_width;
    int32_t ctas;
    int32_t share;               /* circle-schedule pairs per CTA */
} concord_blocked_plan_t;
int concord_blocked_plan(int64_t p, int32_t n_sms, concord_blocked_plan_t* out);

/* Streaming multiprocessors of a device: a caller running k independent fits concurrently
 * (e.g. the cold fits of a lambda path) gives each a solver of n_blocks = SMs / k, on its own
 * stream.  No reference counterpart. */
int concord_device_sm_count(int32_t device, int32_t* out);

int concord_host_alloc(int64_t bytes, void** out);
int concord_host_free(void* ptr);

/* ---- one-shot conveniences ---------------------------------------------- */
int concord_gram_f64(const double* X, int64_t n, int64_t p, double* T_out, int32_t device);
/* center_columns (model.py:182-187) in place on X (n x p row-major, host or device memory per
 * `where`), bitwise numpy's x - x.mean(axis=0). */
int concord_center_columns_f64(double* X, int64_t n, int64_t p, int32_t where, int32_t device);
int concord_pcd_fit(const double* T, int64_t p, double n, const concord_fit_params* prm, double* omega_out,
                    concord_fit_result* res, double* delta_trace, double* objective_trace,
                    double* sweep_seconds, int32_t device);

/* ---- bit-exact reference kernel protocol (host buffers, one sweep) ------- */
/* Bitwise equal to the reference's compiled backend for the same inputs.     */
int concord_pcd_sweep_exact(double* om, const double* t, int64_t p, double n, double shrink,
                            const int64_t* rs, const int64_t* ss, const int64_t* offsets, int64_t nrounds,
                            int32_t device);
int concord_u2_sweep_exact(double* om, const double* t, int64_t p, double n, double shrink, const int64_t* rs,
                           const int64_t* ss, int64_t npairs, int32_t device);
int concord_cd_sweep_exact(double* om, const double* t, int64_t p, double n, double shrink, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* CONCORD_PCD_H */
