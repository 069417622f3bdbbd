// Issue rate of the FMA flavours the fp16 stencil could use, one CTA of W warps on one SM (B200):
//   FFMA (fma.rn.f32), FHFMA (fma.rn.f32.f16: f16 inputs, f32 accumulate), HFMA2 (fma.rn.f16x2),
//   FFMA2 (fma.rn.f32x2).  8 independent chains per thread; reports warp-instructions per cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fma_kinds.cu -o fma_kinds && ./fma_kinds
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int K>
__global__ void bench(float *out, int iters, long long *cyc, uint32_t seed)
{
    float f[8];
    uint32_t h[8];
    unsigned long long d[8];
    for (int i = 0; i < 8; i++) {
        f[i] = (float)(threadIdx.x + i) * 1e-3f;
        h[i] = seed * (i + 1) ^ threadIdx.x;
        d[i] = ((unsigned long long)h[i] << 32) | h[i];
    }
    const uint32_t hm = seed | 0x3c003c00u;
    const float fm = 1.0001f;
    const unsigned long long dm = ((unsigned long long)__float_as_uint(fm) << 32) | __float_as_uint(fm);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (K == 0) f[i] = fmaf(f[i], fm, 0.5f);
            if (K == 1) asm volatile("{.reg .f16 a, b;\nmov.b32 {a, b}, %1;\nfma.rn.f32.f16 %0, a, b, %0;}" : "+f"(f[i]) : "r"(h[i] ^ hm));
            if (K == 2) asm volatile("fma.rn.f16x2 %0, %0, %1, %1;" : "+r"(h[i]) : "r"(hm));
            if (K == 3) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(d[i]) : "l"(dm));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; i++) s += f[i] + __uint_as_float(h[i]) + __uint_as_float((uint32_t)d[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    float *out;
    long long *cyc, hc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8);
    const char *names[4] = {"FFMA", "FHFMA (f32 += f16*f16)", "HFMA2", "FFMA2"};
    const int iters = 4096;
    for (int W : {4, 8, 16}) {
        for (int k = 0; k < 4; k++) {
            for (int rep = 0; rep < 2; rep++) {
                if (k == 0) bench<0><<<1, 32 * W>>>(out, iters, cyc, 0x1234);
                if (k == 1) bench<1><<<1, 32 * W>>>(out, iters, cyc, 0x1234);
                if (k == 2) bench<2><<<1, 32 * W>>>(out, iters, cyc, 0x1234);
                if (k == 3) bench<3><<<1, 32 * W>>>(out, iters, cyc, 0x1234);
            }
            cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
            const double winst = (double)iters * 8 * W;
            printf("W=%2d %-24s %.2f warp-instr/cycle/SM\n", W, names[k], winst / hc);
        }
    }
    return 0;
}
