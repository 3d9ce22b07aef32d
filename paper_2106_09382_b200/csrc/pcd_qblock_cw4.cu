// The temporally blocked kernel with 4 chain warps (pcd_qblock_impl.cuh), the roles aligned to
// warp groups so setmaxnreg hands registers between them: chain warps 88, apply warps 136.
#define QB_NS qb4
#define QB_NS_CHAIN_WARPS 4
#define QB_NS_REGS_CHAIN 88
#define QB_NS_REGS_APPLY 136
#include "pcd_qblock_impl.cuh"
