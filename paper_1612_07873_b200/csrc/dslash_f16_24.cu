// Instantiation unit: coarse-Dslash kernels for storage CD_FP16, Nvec = 24.
#include "dslash_impl.cuh"
CD_INSTANTIATE(CD_FP16, 24, f16_24)
