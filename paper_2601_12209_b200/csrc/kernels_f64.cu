#define DFFT_REAL double
#define DFFT_LOOKUP lookup_kernel_f64
#include "kernels_inst.cuh"
