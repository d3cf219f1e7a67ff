// Element-kernel instantiations for mode M_GRAD_APPLY.
#define HPG_MODE hpg::M_GRAD_APPLY
#define HPG_WARP_LIST HPG_W(1,1) HPG_W(1,2) HPG_W(1,3) HPG_W(2,2) HPG_W(2,3) HPG_W(2,4)
#include "hpg_mode_impl.cuh"
