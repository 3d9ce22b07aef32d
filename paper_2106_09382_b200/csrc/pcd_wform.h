// Internal C++ interface of the W-form persistent kernel (not the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define WFORM_THREADS 512
#define WFORM_CHAIN_WARPS 4     // warps 0..3: publish / closed forms / grid barrier (the colour chain)
#define WFORM_PAIR_CAP 1024     // delta-list pairs staged in shared memory per apply chunk
#define WFORM_SHARE_MIN 1       // closed forms per share CTA per colour (fewer, longer delta-list segments)
#define WFORM_BATCH 8           // colour phases one apply batch may cover
#define WFORM_STAGE_SLOTS 5     // publish stages in flight (shared memory ring)
#define WFORM_MAX_LAG 8         // max phases the apply warps may trail the chain
#define WFORM_MAX_BLOCKS 1024

namespace concord {

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
    double2* pub;   // 3 * p rotating publish buffers (global phase mod 3)
    double* dring;  // [rd][p] per-row delta of each recent phase (0.0 where the pair did not move)
    double2* diagd; // [nblk][p] (delta, new) of the last diagonal step, per CTA
    double n;       // sample count (GramMatrix.n)
    double shrink;  // n * lam (solver.py:285)
    double delta_tol;
    int max_iter;
    int want_trace;
    int lmax;       // lag cap of the apply warps behind the chain (<= WFORM_MAX_LAG, <= m)
    int rd;         // dring slots (>= lmax + 3)
    int rl;         // delta-list ring slots (>= lmax + 4)
    unsigned long long* bar;
    double* rec_delta;              // [max_iter]
    double* rec_obj;                // [max_iter][nblk][3]: <W,Om> part, sum_{i<j}|om|, sum log om_ii
    unsigned long long* rec_time;   // [max_iter + 1] globaltimer ns
    long long* rec_nnz;             // [max_iter] non-zero off-diagonal deltas per sweep (zeroed by host)
    unsigned long long* rec_dmax;   // [max_iter] max |off-diagonal delta| per sweep, double bits (zeroed)
    int share;                      // pairs per share CTA per colour
    int nsh;                        // CTAs that evaluate closed forms (ceil(half / share))
    int stage_ahead;                // publishes staged beyond the chain's phase
    int2* list_rs;                  // [rl][nblk][share] non-zero pairs of a colour, per CTA segment
    double2* list_dn;               // [rl][nblk][share] (delta, new value)
    int* list_cnt;                  // [rl][nblk] segment lengths
    int* status;                    // [0] iterations, [1] converged
    unsigned long long* prof;       // optional [16] cycle counters (CTA 0), or NULL
};

// Lag cap for a slab width (bounded by the stage ring's shared memory) and m.
int wform_lag_cap(int w, int m);
size_t wform_smem_bytes(int w, int p, int nblk, int lmax);

cudaError_t launch_pcd_wform(const WformArgs& args, int nblk, cudaStream_t st);
cudaError_t wform_max_blocks(int w, int p, int* max_blocks);
cudaError_t launch_pack_slabs(const double* src, long long ld, double* dst, int p, int w, int nblk,
                              cudaStream_t st);
cudaError_t launch_unpack_slabs(const double* src, double* dst, int p, int w, cudaStream_t st);
cudaError_t launch_slab_diag(const double* slab, double* diag, int p, int w, cudaStream_t st);
cudaError_t launch_slab_identity(double* slab, int p, int w, int nblk, cudaStream_t st);
cudaError_t launch_slab_edge_count(const double* slab, int p, int w, int nblk, unsigned long long* out,
                                   cudaStream_t st);
cudaError_t launch_wform_init_csr(const int* rowptr, const int* colidx, const double* vals, const double* Tslab,
                                  double* Wslab, int p, int w, int nblk, cudaStream_t st);

// Exact (direct-form) reference-protocol sweeps, pcd_exact.cu.
cudaError_t launch_pcd_sweep_exact(double* om, const double* t, int p, double n, double shrink,
                                   const long long* rs, const long long* ss, const long long* offsets,
                                   int nrounds, unsigned long long* bar, cudaStream_t st);
cudaError_t launch_u2_sweep_exact(double* om, const double* t, int p, double n, double shrink,
                                  const long long* rs, const long long* ss, long long npairs, cudaStream_t st);
cudaError_t launch_cd_sweep_exact(double* om, const double* t, int p, double n, double shrink, cudaStream_t st);

// FP64 DMMA Gram / GEMM, gram.cu.  T = X^T X (X: n x p row-major, leading dim ldx).
// out_mode 0: row-major p x p (ld = p); 1: slab-major with width w.
cudaError_t launch_gram_f64(const double* X, long long n, int p, long long ldx, double* out, int out_mode, int w,
                            cudaStream_t st);

}  // namespace concord
