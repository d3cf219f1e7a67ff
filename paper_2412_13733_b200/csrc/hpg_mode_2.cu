// Element-kernel instantiations for mode M_OBST_CACHED.
#define HPG_MODE hpg::M_OBST_CACHED
#define HPG_WARP_LIST HPG_W(1,1) HPG_W(1,2) HPG_W(1,3) HPG_W(1,4) HPG_W(2,2) HPG_W(2,3) HPG_W(2,4) HPG_W(2,5)
#define HPG_WSPLIT_LIST HPG_WS(1,2) HPG_WS(1,3)
#include "hpg_mode_impl.cuh"
