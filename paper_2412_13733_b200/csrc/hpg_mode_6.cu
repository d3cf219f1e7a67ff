// Element-kernel instantiations for mode M_VALUES.
#define HPG_MODE hpg::M_VALUES
#define HPG_WARP_LIST 
#include "hpg_mode_impl.cuh"
