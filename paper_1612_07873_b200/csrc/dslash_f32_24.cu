// Instantiation unit: coarse-Dslash kernels for storage CD_FP32, Nvec = 24.
#include "dslash_impl.cuh"
CD_INSTANTIATE(CD_FP32, 24, f32_24)
