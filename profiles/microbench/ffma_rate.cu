// FP32 MAC issue rate on one SM for the cluster-push chain's inner loop shapes (B200, sm_100a):
// complex MACs of register-resident link chunks with vector chunks from shared memory, as
//   F: 4 x FFMA per complex (cmac2),  P: 2 x FFMA2 (scalar broadcast) per complex (cmac2x),
// with W warps in one CTA; reports cycles per complex MAC per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma_rate.cu -o ffma_rate && ./ffma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cmac2(const uint4 &a, const uint4 &b, float &re, float &im)
{
    float ar0 = __uint_as_float(a.x), ai0 = __uint_as_float(a.y), ar1 = __uint_as_float(a.z), ai1 = __uint_as_float(a.w);
    float br0 = __uint_as_float(b.x), bi0 = __uint_as_float(b.y), br1 = __uint_as_float(b.z), bi1 = __uint_as_float(b.w);
    re = fmaf(ar0, br0, re); im = fmaf(ar0, bi0, im); re = fmaf(-ai0, bi0, re); im = fmaf(ai0, br0, im);
    re = fmaf(ar1, br1, re); im = fmaf(ar1, bi1, im); re = fmaf(-ai1, bi1, re); im = fmaf(ai1, br1, im);
}
__device__ __forceinline__ void cmac2x(const uint4 &a, const uint4 &b, unsigned long long &A, unsigned long long &B)
{
    asm("{\n.reg .b64 l0, l1, v0, v1, i0, i1;\n"
        "mov.b64 l0, {%2, %2};\nmov.b64 i0, {%3, %3};\nmov.b64 v0, {%6, %7};\n"
        "fma.rn.f32x2 %0, l0, v0, %0;\nfma.rn.f32x2 %1, i0, v0, %1;\n"
        "mov.b64 l1, {%4, %4};\nmov.b64 i1, {%5, %5};\nmov.b64 v1, {%8, %9};\n"
        "fma.rn.f32x2 %0, l1, v1, %0;\nfma.rn.f32x2 %1, i1, v1, %1;\n}"
        : "+l"(A), "+l"(B) : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w));
}

constexpr int NC = 24;   // link chunks per thread (48 complex MACs per pass)

template <int MODE>   // 0: FFMA, 2 accumulators; 1: FFMA, 4 accumulators; 2: FFMA2
__global__ void __launch_bounds__(384, 1) bench(const uint4 *L, float *out, int iters, long long *cyc)
{
    __shared__ uint4 vs[64];
    if (threadIdx.x < 64) vs[threadIdx.x] = L[threadIdx.x + 1000];
    __syncthreads();
    uint4 l[NC];
#pragma unroll
    for (int i = 0; i < NC; i++) l[i] = L[(threadIdx.x * NC + i) & 4095];
    const int d = threadIdx.x & 7;
    float re = 0, im = 0, re2 = 0, im2 = 0;
    unsigned long long A = 0, B = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const uint4 *v = vs + ((it & 1) * 32);
#pragma unroll
        for (int c = 0; c < NC; c++) {
            uint4 vv;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(vv.x), "=r"(vv.y), "=r"(vv.z), "=r"(vv.w)
                         : "r"((uint32_t)__cvta_generic_to_shared(v + ((d + 8 * c) & 31))));
            if (MODE == 0) cmac2(l[c], vv, re, im);
            else if (MODE == 1) { if (c & 1) cmac2(l[c], vv, re2, im2); else cmac2(l[c], vv, re, im); }
            else cmac2x(l[c], vv, A, B);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = re + im + re2 + im2 + __uint_as_float((unsigned)A) + __uint_as_float((unsigned)(B >> 32));
}

int main()
{
    uint4 *L; float *out; long long *cyc;
    cudaMalloc(&L, 8192 * 16); cudaMemset(L, 0, 8192 * 16);
    cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
    const int iters = 2000;
    for (int mode = 0; mode < 3; mode++)
        for (int w : {4, 8, 12}) {
            void (*k)(const uint4 *, float *, int, long long *) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : bench<2>;
            k<<<1, 32 * w>>>(L, out, 10, cyc);
            k<<<1, 32 * w>>>(L, out, iters, cyc);
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double cmacs_per_smsp = (double)iters * NC * 2 * w / 4.0;   // complex MACs per SMSP
            // per SMSP: cmacs_per_smsp warp-level complex MACs = 4 FFMA (or 2 FFMA2) warp instructions each
            printf("mode %s warps %2d: %.3f cycles per warp complex MAC per SMSP = %.1f real FMA/clk/SM\n",
                   mode == 0 ? "FFMA  2acc" : mode == 1 ? "FFMA  4acc" : "FFMA2     ", w, c / cmacs_per_smsp,
                   4.0 * 32 * 4 * cmacs_per_smsp / c);
        }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
