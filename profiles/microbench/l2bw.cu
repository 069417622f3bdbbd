// L2 -> SM read bandwidth microbenchmark (roofline denominator for L2-bound kernels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu && ./l2bw
// (a) LDG.128: every CTA streams the whole L2-resident buffer `passes` times (grid-stride,
//     16 B per thread per load, 8 loads in flight per thread);
// (b) TMA bulk: one thread per CTA issues cp.async.bulk copies of 16 KB chunks into a 6-stage
//     smem ring (mbarrier complete_tx), the pattern of the multi-RHS producer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void ldg_kernel(const uint4 *__restrict__ buf, size_t n16, int passes, unsigned *out)
{
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; p++) {
        size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x + (size_t)p * 977 * blockDim.x;
        for (size_t k = 0; k < n16 / stride; k += 8) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = __ldcg(&buf[(i + (k + u) * stride) % n16]);
#pragma unroll
            for (int u = 0; u < 8; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned ph)
{
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b)),
                 "r"(ph)
                 : "memory");
}

template <int S, int CH>
__global__ void tma_kernel(const unsigned char *buf, size_t bytes, int chunks_per_cta, unsigned *out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm);
    unsigned char *ring = sm + 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const size_t nch = bytes / CH;
    for (int c = 0; c < chunks_per_cta; c++) {
        const int s = c % S;
        if (c >= S) mbar_wait(&full[s], ((c / S) - 1) & 1);
        const size_t ch = ((size_t)blockIdx.x * 7919 + (size_t)c * 131) % nch;
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(ring + s * CH)),
                     "l"(buf + ch * CH), "r"(CH), "r"(bar)
                     : "memory");
    }
    for (int c = chunks_per_cta - S; c < chunks_per_cta; c++) mbar_wait(&full[c % S], (c / S) & 1);
    if (ring[5] == 0x7f) out[1] = 1;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *out;
    cudaMalloc(&out, 16);
    printf("{");
    for (size_t mb : {32, 64, 96}) {
        const size_t bytes = mb << 20;
        unsigned char *buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        // (a) LDG
        const int passes = 4, grid = sms * 4, block = 512;
        ldg_kernel<<<grid, block>>>((const uint4 *)buf, bytes / 16, 1, out);
        cudaEventRecord(e0);
        ldg_kernel<<<grid, block>>>((const uint4 *)buf, bytes / 16, passes, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ldg = (double)((bytes / 16 / ((size_t)grid * block) + 7) / 8 * 8) * (size_t)grid * block * 16 * passes / (ms * 1e-3) / 1e9;
        // (b) TMA, 1 CTA per SM, (stages x chunk) rings
        auto run = [&](auto kern, int S, int CH) {
            const int cpc = (int)(((size_t)256 << 20) / CH);
            const int smem = 128 + S * CH;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            kern<<<sms, 32, smem>>>(buf, bytes, 64, out);
            cudaEventRecord(e0);
            kern<<<sms, 32, smem>>>(buf, bytes, cpc, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            return (double)sms * cpc * CH / (t * 1e-3) / 1e9;
        };
        const double t1 = run(tma_kernel<6, 16384>, 6, 16384);
        const double t2 = run(tma_kernel<5, 33792>, 5, 33792);
        const double t3 = run(tma_kernel<3, 33792>, 3, 33792);
        const double t4 = run(tma_kernel<12, 8192>, 12, 8192);
        printf("%s\"%zuMB\": {\"ldg_GBs\": %.1f, \"tma_6x16K\": %.1f, \"tma_5x33K\": %.1f, \"tma_3x33K\": %.1f, \"tma_12x8K\": %.1f}",
               mb == 32 ? "" : ", ", mb, ldg, t1, t2, t3, t4);
        cudaFree(buf);
    }
    printf(", \"sms\": %d, \"err\": \"%s\"}\n", sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
