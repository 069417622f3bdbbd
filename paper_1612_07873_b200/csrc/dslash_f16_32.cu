// Instantiation unit: coarse-Dslash kernels for storage CD_FP16, Nvec = 32.
#include "dslash_impl.cuh"
CD_INSTANTIATE(CD_FP16, 32, f16_32)
