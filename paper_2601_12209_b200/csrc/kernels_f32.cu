#define DFFT_REAL float
#define DFFT_LOOKUP lookup_kernel_f32
#include "kernels_inst.cuh"
