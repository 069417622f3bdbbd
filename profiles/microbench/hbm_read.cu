// HBM read-only streaming bandwidth (the achievable denominator for the read-dominated stencil):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_read hbm_read.cu && ./hbm_read
// Reads a buffer much larger than L2 once per launch with 128-bit non-allocating loads
// (ld.global.nc.L1::no_allocate, the links' load path), grid = k x 148 CTAs, 8 loads in
// flight per thread; also a 680 MB buffer (one 8^4 fp32 link set) back to back with
// launch gaps included, i.e. the per-apply read the 8^4 kernels do.  Best of 20 launches.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_stream(const void *p)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__global__ void __launch_bounds__(512) rd(const uint4 *__restrict__ buf, size_t n16, unsigned *out)
{
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = ld_stream(&buf[i + u * stride]);
#pragma unroll
        for (int u = 0; u < 8; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        uint4 v = ld_stream(&buf[i]);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *out;
    cudaMalloc(&out, 4);
    for (size_t bytes : {(size_t)680 << 20, (size_t)4 << 30}) {
        uint4 *buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        const size_t n16 = bytes / 16;
        for (int k : {2, 4, 8}) {
            for (int threads : {256, 512}) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                float best = 1e30f;
                for (int r = 0; r < 20; r++) {
                    cudaEventRecord(e0);
                    rd<<<k * sms, threads>>>(buf, n16, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("read %6.0f MB  grid %d x %d SMs, %3d threads: %.1f us  %.0f GB/s\n", bytes / 1048576.0, k, sms,
                       threads, best * 1e3, bytes / (best * 1e-3) / 1e9);
            }
        }
        cudaFree(buf);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
