// ipc_flag_probe.cu -- can two processes on ONE GPU hand data to each other through CUDA IPC
// memory with a device-side release/acquire flag (no host sync), and how long does a round take?
// (Round-2 design question for the peer-push halo transport.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o /tmp/ipcp.so ipc_flag_probe.cu
// driven by profiles/microbench/ipc_flag_probe.py (torch.multiprocessing, 2 ranks, cuda:0).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>

__global__ void put_signal(const int *src, int *peer_dst, int n, unsigned long long *peer_flag, unsigned long long epoch)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) peer_dst[i] = src[i] + (int)epoch;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        atomicAdd(peer_flag, 1ull);
    }
}

__global__ void wait_read(const int *buf, int n, const unsigned long long *flag, unsigned long long target, int *out,
                          int *timeout)
{
    if (threadIdx.x == 0) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
            if (v >= target) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 5000000000ull) {
                atomicExch(timeout, 1);
                break;
            }
        }
    }
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = buf[i];
}

extern "C" {
int p_malloc(size_t b, void **p)
{
    cudaError_t e = cudaMalloc(p, b);
    if (e == cudaSuccess) e = cudaMemset(*p, 0, b);
    return (int)e;
}
int p_sync() { return (int)cudaDeviceSynchronize(); }
int p_ipc_handle(void *ptr, unsigned char out[64])
{
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
    memcpy(out, &h, 64);
    return (int)e;
}
int p_ipc_open(const unsigned char in[64], void **out)
{
    cudaIpcMemHandle_t h;
    memcpy(&h, in, 64);
    return (int)cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
}
int p_put(const int *src, int *peer_dst, int n, unsigned long long *peer_flag, unsigned long long epoch, void *s)
{
    put_signal<<<4, 256, 0, (cudaStream_t)s>>>(src, peer_dst, n, peer_flag, epoch);
    return (int)cudaGetLastError();
}
int p_wait(const int *buf, int n, const unsigned long long *flag, unsigned long long target, int *out, int *timeout,
           void *s)
{
    wait_read<<<4, 256, 0, (cudaStream_t)s>>>(buf, n, flag, target, out, timeout);
    return (int)cudaGetLastError();
}
}
