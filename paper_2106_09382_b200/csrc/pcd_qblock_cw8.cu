// The temporally blocked kernel with 8 chain warps (pcd_qblock_impl.cuh), the roles aligned to
// warp groups so setmaxnreg hands registers between them: chain warps 96, apply warps 160.
#define QB_NS qb8
#define QB_NS_CHAIN_WARPS 8
#define QB_NS_REGS_CHAIN 96
#define QB_NS_REGS_APPLY 160
#include "pcd_qblock_impl.cuh"
