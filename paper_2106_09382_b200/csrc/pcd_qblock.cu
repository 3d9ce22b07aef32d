// The temporally blocked kernel, default variant (6 chain warps, one register budget), and the
// host-side dispatch over the chain-warp variants (pcd_qblock_cw4.cu: apply-heavy, for the dense
// fits; pcd_qblock_cw8.cu: chain-heavy, for sparse fits on small lanes).  The kernel itself is
// pcd_qblock_impl.cuh.
#define QB_NS qb6
#define QB_NS_CHAIN_WARPS 6
#define QB_NS_REGS_CHAIN 0
#define QB_NS_REGS_APPLY 0
#include "pcd_qblock_impl.cuh"

namespace concord {

int qblock_cellcap(int share, int D) { return 2 * D * (share + 2 * (D - 1)) + 2 * share + 8; }

int qblock_rmax(int share, int D) { return share + 2 * (D - 1) + 2; }

bool qblock_variant_ok(int chain_warps) { return chain_warps == 4 || chain_warps == 6 || chain_warps == 8; }

size_t qblock_smem_bytes(int chain_warps, int p, int nblk, int share, int D, int tdiag_smem, int nbuf,
                         int ring_stages) {
    if (chain_warps == 4) return qb4::smem_bytes(p, nblk, share, D, tdiag_smem, nbuf, ring_stages);
    if (chain_warps == 8) return qb8::smem_bytes(p, nblk, share, D, tdiag_smem, nbuf, ring_stages);
    return qb6::smem_bytes(p, nblk, share, D, tdiag_smem, nbuf, ring_stages);
}

int qblock_colour_warps(int chain_warps, int share, int D) {
    if (chain_warps == 4) return qb4::colour_warps_host(share, D);
    if (chain_warps == 8) return qb8::colour_warps_host(share, D);
    return qb6::colour_warps_host(share, D);
}

cudaError_t qblock_reserve_smem(int chain_warps, size_t smem) {
    if (chain_warps == 4) return qb4::reserve_smem(smem);
    if (chain_warps == 8) return qb8::reserve_smem(smem);
    return qb6::reserve_smem(smem);
}

cudaError_t launch_pcd_qblock(const QbArgs& args, int nblk, cudaStream_t st) {
    if (args.chain_warps == 4) return qb4::launch(args, nblk, st);
    if (args.chain_warps == 8) return qb8::launch(args, nblk, st);
    return qb6::launch(args, nblk, st);
}

}  // namespace concord
