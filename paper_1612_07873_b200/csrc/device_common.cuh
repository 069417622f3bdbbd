// device_common.cuh -- sm_100a device helpers shared by the coarse-Dslash kernels.
// (PTX wrappers for 128-bit streaming loads, cp.async.bulk + mbarrier, PDL, FHFMA,
//  fast integer division, and per-precision record geometry.)
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

#include "cd_internal.h"

namespace cd {

// ------------------------------------------------------------------ record geometry
// One 16-byte "chunk" = 2 complex (fp32) or 4 complex (fp16).  A matrix row of N complex
// is N/2 (fp32) or N/4 (fp16) chunks; D lanes share a row (lane d reads chunks
// d, d+D, d+2D, ...), R = 32/D rows per warp, C = N/16 chunks per lane per row.
template <cd_precision P, int NV>
struct Cfg {
    static constexpr int N = 2 * NV;
    static constexpr bool F16 = (P == CD_FP16);
    static constexpr int CPC = F16 ? 4 : 2;                    // complex per 16-B chunk
    static constexpr int ROWB = F16 ? 4 * N : 8 * N;           // bytes per matrix row
    static constexpr int MREC = F16 ? 4 * N * N + 16 : 8 * N * N;  // matrix record bytes
    static constexpr int VREC = F16 ? 4 * N + 16 : 8 * N;      // vector record bytes
    static constexpr int MSCALE = 4 * N * N;                   // fp16: scale offset in matrix record
    static constexpr int VSCALE = 4 * N;                       // fp16: scale offset in vector record
    static constexpr int D = F16 ? 4 : 8;                      // lanes per row
    static constexpr int R = 32 / D;                           // rows per warp
    static constexpr int C = N / 16;                           // chunks per lane per row
    static constexpr int VCH = VREC / 16;                      // 16-B chunks per vector record
    static_assert(C * D * CPC == N, "chunk geometry");
};

// ------------------------------------------------------------------ memory ops
__device__ __forceinline__ uint4 ld_stream(const void *p)
{   // links: read once per apply -> bypass L1
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_nc(const void *p)
{
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_nc_f32(const void *p)
{
    float r;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
// 128-bit shared-memory load as a plain C++ access (not volatile asm): the compiler may batch and
// hoist these loads (they only move within barrier-delimited regions), which hides their latency
// when several chunks feed independent FMA chains.
__device__ __forceinline__ uint4 lds128(const void *p) { return *reinterpret_cast<const uint4 *>(p); }

// ------------------------------------------------------------------ PDL (griddepcontrol)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------ mbarrier + bulk copy
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)), "l"(src), "r"(bytes),
          "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy: evict_first for streamed-once data,
// evict_last for data re-read by other CTAs)
__device__ __forceinline__ uint64_t l2_policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)), "l"(src), "r"(bytes),
          "r"((uint32_t)__cvta_generic_to_shared(bar)), "l"(policy) : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (no shared-memory destination, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 4-byte asynchronous shared-memory store whose completion is counted (4 tx bytes) on an
// mbarrier: a value delivered exactly like TMA data, ordered by the barrier's phase.
__device__ __forceinline__ void st_async_u32(void *dst_smem, uint32_t v, uint64_t *bar)
{
    // st.async addresses live in the shared::cluster window: map this CTA's own addresses there
    uint32_t rank, d, b;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"((uint32_t)__cvta_generic_to_shared(dst_smem)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b) : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(d), "r"(v), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void bar_named(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ arithmetic
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f)
{
    uint32_t hi = __umulhi(n, f.m);
    return (hi + n) >> f.s;   // n < 2^31 -> no overflow
}

// fp32 complex MAC of one 16-B chunk pair: (a0, a1) . (b0, b1)
__device__ __forceinline__ void cmac2(const uint4 &a, const uint4 &b, float &re, float &im)
{
    float ar0 = __uint_as_float(a.x), ai0 = __uint_as_float(a.y), ar1 = __uint_as_float(a.z), ai1 = __uint_as_float(a.w);
    float br0 = __uint_as_float(b.x), bi0 = __uint_as_float(b.y), br1 = __uint_as_float(b.z), bi1 = __uint_as_float(b.w);
    re = fmaf(ar0, br0, re);
    im = fmaf(ar0, bi0, im);
    re = fmaf(-ai0, bi0, re);
    im = fmaf(ai0, br0, im);
    re = fmaf(ar1, br1, re);
    im = fmaf(ar1, bi1, im);
    re = fmaf(-ai1, bi1, re);
    im = fmaf(ai1, br1, im);
}

// fp32 complex MAC of one 16-B chunk pair on the packed FP32 pipe (SASS FFMA2 with a scalar
// broadcast operand): A += lr * (vr, vi), B += li * (vr, vi) for both complex of the chunk;
// the complex result is (A.x - B.y, A.y + B.x).  Two FFMA2 per complex MAC instead of four FFMA,
// and the vector pair is read once (reuse) for both.
__device__ __forceinline__ void cmac2x(const uint4 &a, const uint4 &b, unsigned long long &A, unsigned long long &B)
{
    asm("{\n.reg .b64 l0, l1, v0, v1, i0, i1;\n"
        "mov.b64 l0, {%2, %2};\n"
        "mov.b64 i0, {%3, %3};\n"
        "mov.b64 v0, {%6, %7};\n"
        "fma.rn.f32x2 %0, l0, v0, %0;\n"
        "fma.rn.f32x2 %1, i0, v0, %1;\n"
        "mov.b64 l1, {%4, %4};\n"
        "mov.b64 i1, {%5, %5};\n"
        "mov.b64 v1, {%8, %9};\n"
        "fma.rn.f32x2 %0, l1, v1, %0;\n"
        "fma.rn.f32x2 %1, i1, v1, %1;\n}"
        : "+l"(A), "+l"(B) : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w));
}

// fp16 complex MAC of one complex pair held as half2 {re, im} words, fp32 accumulate:
// one FHFMA (fma.rn.f32.f16) per real product; no conversions (SURVEY §0 probe).
//   ra += lr*vr, rb += li*vi, ia += lr*vi, ib += li*vr   ->  re = ra - rb, im = ia + ib
__device__ __forceinline__ void hmac1(uint32_t l, uint32_t v, float &ra, float &rb, float &ia, float &ib)
{
    asm("{\n.reg .f16 lr, li, vr, vi;\n"
        "mov.b32 {lr, li}, %4;\n"
        "mov.b32 {vr, vi}, %5;\n"
        "fma.rn.f32.f16 %0, lr, vr, %0;\n"
        "fma.rn.f32.f16 %1, li, vi, %1;\n"
        "fma.rn.f32.f16 %2, lr, vi, %2;\n"
        "fma.rn.f32.f16 %3, li, vr, %3;\n}"
        : "+f"(ra), "+f"(rb), "+f"(ia), "+f"(ib) : "r"(l), "r"(v));
}
__device__ __forceinline__ void hmac4(const uint4 &a, const uint4 &b, float &ra, float &rb, float &ia, float &ib)
{
    hmac1(a.x, b.x, ra, rb, ia, ib);
    hmac1(a.y, b.y, ra, rb, ia, ib);
    hmac1(a.z, b.z, ra, rb, ia, ib);
    hmac1(a.w, b.w, ra, rb, ia, ib);
}

// tau3 on an input chunk (components j >= Nvec flip sign; R5/R6)
template <bool F16>
__device__ __forceinline__ uint4 neg_chunk(uint4 v)
{
    const uint32_t m = F16 ? 0x80008000u : 0x80000000u;
    v.x ^= m; v.y ^= m; v.z ^= m; v.w ^= m;
    return v;
}

// Thread-block cluster helpers (DSMEM reads + full-cluster barrier).
__device__ __forceinline__ unsigned cluster_rank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint4 ld_dsmem(const void *local_ptr, unsigned cta)
{
    uint32_t la = (uint32_t)__cvta_generic_to_shared(local_ptr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(cta));
    uint4 v;
    asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ra)
                 : "memory");
    return v;
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Site decode (Listing 2, x0 fastest) with host-computed magic numbers.
__device__ __forceinline__ void decode(const KGeom &g, int s, int x[4])
{
    uint32_t t1 = fdiv((uint32_t)s, g.fd[0]);
    x[0] = s - (int)t1 * g.L[0];
    uint32_t t2 = fdiv(t1, g.fd[1]);
    x[1] = (int)t1 - (int)t2 * g.L[1];
    uint32_t t3 = fdiv(t2, g.fd[2]);
    x[2] = (int)t2 - (int)t3 * g.L[2];
    x[3] = (int)t3;
}
__device__ __forceinline__ int encode(const KGeom &g, const int x[4])
{
    return ((x[3] * g.L[2] + x[2]) * g.L[1] + x[1]) * g.L[0] + x[0];
}
// x[mu] for a run-time mu without dynamic register indexing (keeps x in registers).
__device__ __forceinline__ int sel4(const int v[4], int mu)
{
    return mu == 0 ? v[0] : (mu == 1 ? v[1] : (mu == 2 ? v[2] : v[3]));
}
// Neighbour of x through hop k (k = 2mu + dir; k = 8 -> x), periodic (R10):
// s +- stride(mu), with the wrap folded in -- no re-encode, no dynamic indexing.
__device__ __forceinline__ int neighbour(const KGeom &g, const int x[4], int s, int k)
{
    if (k == 8) return s;
    const int mu = k >> 1;
    const int L = sel4(g.L, mu);
    const int xm = sel4(x, mu);
    const int stride = mu == 0 ? 1 : (mu == 1 ? g.L[0] : (mu == 2 ? g.L[0] * g.L[1] : g.L[0] * g.L[1] * g.L[2]));
    if (k & 1) return xm == 0 ? s + (L - 1) * stride : s - stride;
    return xm == L - 1 ? s - (L - 1) * stride : s + stride;
}
// Is hop k of x remote (its neighbour lives on another rank / in the halo)?
__device__ __forceinline__ bool remote_hop(const KGeom &g, const int x[4], int k)
{
    if (k == 8) return false;
    const int mu = k >> 1;
    if (!((g.split >> mu) & 1)) return false;
    const int xm = sel4(x, mu);
    return (k & 1) ? (xm == 0) : (xm == sel4(g.L, mu) - 1);
}

// Hop order inside a site: X first, then k = 0..7 (fixed term order, R11).
__device__ __forceinline__ int kseq(int i) { return i == 0 ? 8 : i - 1; }

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// Peer transport: after a CTA has stored its part of a halo block into the
// receiver's window, bump the receiver's arrival counter once (release, system scope; the
// CTA barrier orders every thread's stores before thread 0's fence).
__device__ __forceinline__ void signal_block(unsigned long long *flag)
{
    __syncthreads();
    if (threadIdx.x == 0 && flag) {
        __threadfence_system();
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(flag) : "memory");
    }
}

}  // namespace cd
