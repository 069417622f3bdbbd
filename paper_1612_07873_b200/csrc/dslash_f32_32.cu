// Instantiation unit: coarse-Dslash kernels for storage CD_FP32, Nvec = 32.
#include "dslash_impl.cuh"
CD_INSTANTIATE(CD_FP32, 32, f32_32)
