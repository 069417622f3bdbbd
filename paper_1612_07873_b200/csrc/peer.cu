// peer.cu -- device side of the peer (CUDA IPC / NVLink) halo transport.
//
// The paper moves the coarse halo through the host: pack -> D2H -> MPI -> H2D, with no
// overlap (§6.5).  Here the ranks map each other's receive windows (CUDA IPC;
// over NVLink / NVSwitch between GPUs, or the same device for several processes on one GPU),
// the halo pack kernel stores the face records straight into the neighbour's window and bumps
// an arrival counter there (device_common.cuh signal_block), and the receiver's stream runs
// the wait kernel below before its halo-term kernel.  No host synchronisation, no NCCL.
//
// Counters are monotonic: every exchange adds kPutCtas to each block's counter, so exchange e
// (1-based, the same sequence on every rank because applies are collective) has landed when
// the counter reaches kPutCtas * e.  Each counter has exactly one writer (the rank that sends
// that block), so contributions of different senders never alias.
#include <cuda_runtime.h>

#include "cd_internal.h"
#include "device_common.cuh"

namespace cd {

__global__ void peer_wait_kernel(PeerWait w)
{
    const int b = threadIdx.x;
    if (b < 8 && ((w.mask >> b) & 1)) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(w.flag + b) : "memory");
            if (v >= w.target) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > w.timeout_ns) {
                atomicExch_system(w.err, 1);   // surfaces at the next call on this context
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
}

cudaError_t launch_peer_wait(const PeerWait &w, cudaStream_t s)
{
    if (!w.mask) return cudaSuccess;
    count_launch();
    peer_wait_kernel<<<1, 32, 0, s>>>(w);
    return cudaGetLastError();
}

struct Blocks {
    const unsigned char *src[4][2];
    unsigned char *dst[4][2];
    int64_t len[4][2];
};

// blockIdx.y = (mu, blk) index 2mu+blk over the 8 possible blocks (blocks not in the mask exit)
__global__ void put_blocks_kernel(Blocks b, PackDst d, unsigned mask, int signal)
{
    const int id = blockIdx.y, mu = id >> 1, blk = id & 1;
    if (!((mask >> id) & 1)) return;   // uniform per CTA: no barrier is skipped by part of a CTA
    const unsigned char *src = b.src[mu][blk];
    unsigned char *dst = b.dst[mu][blk];
    const int64_t n16 = b.len[mu][blk] / 16;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    if (signal) signal_block(d.flag[mu][blk]);
}

cudaError_t launch_peer_put(const unsigned char *const src[4][2], const int64_t len[4][2], unsigned mask,
                            const PackDst &d, cudaStream_t s)
{
    Blocks b{};
    for (int mu = 0; mu < 4; mu++)
        for (int k = 0; k < 2; k++) {
            b.src[mu][k] = src[mu][k];
            b.dst[mu][k] = d.dst[mu][k];
            b.len[mu][k] = len[mu][k];
        }
    count_launch();
    put_blocks_kernel<<<dim3(kPutCtas, 8), 256, 0, s>>>(b, d, mask, 1);
    return cudaGetLastError();
}

cudaError_t launch_copy_blocks(const unsigned char *const src[4][2], unsigned char *const dst[4][2],
                               const int64_t len[4][2], unsigned mask, cudaStream_t s)
{
    Blocks b{};
    for (int mu = 0; mu < 4; mu++)
        for (int k = 0; k < 2; k++) {
            b.src[mu][k] = src[mu][k];
            b.dst[mu][k] = dst[mu][k];
            b.len[mu][k] = len[mu][k];
        }
    PackDst none{};
    count_launch();
    put_blocks_kernel<<<dim3(kPutCtas, 8), 256, 0, s>>>(b, none, mask, 0);
    return cudaGetLastError();
}

}  // namespace cd
