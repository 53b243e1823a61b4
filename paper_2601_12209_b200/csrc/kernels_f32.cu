#define DFFT_REAL float
#define DFFT_LOOKUP lookup_kernel_f32
#define DFFT_LOOKUP_FUSED lookup_fused_xy_f32
#include "kernels_inst.cuh"
