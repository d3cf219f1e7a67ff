// Element-kernel instantiations for mode M_GRAD_RES.
#define HPG_MODE hpg::M_GRAD_RES
#define HPG_WARP_LIST HPG_W(1,1) HPG_W(1,2) HPG_W(1,3) HPG_W(2,2) HPG_W(2,3) HPG_W(2,4)
#define HPG_WSPLIT_LIST HPG_WS(3,5) HPG_WS(3,7)
#include "hpg_mode_impl.cuh"
