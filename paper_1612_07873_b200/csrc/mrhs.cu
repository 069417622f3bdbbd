// mrhs.cu -- multi right-hand-side coarse Dslash on the 5th-generation tensor cores (tcgen05).
//
// SURVEY NEXT-1 (the paper's "multi-right-hand-side MG", §9): with n_rhs vectors
// the per-site work becomes a small GEMM, so tensor cores finally apply.  For one site x and
// one hop k, with B = the stored fp16 link matrix L_k(x) read as a K-major operand (row i =
// output colour-spin, K index = 2j + {re,im}) and A = the 128 right-hand sides' neighbour
// vectors (row r = rhs, same K index):
//
//     A[r][2j]   =  v_r(nbr_k)_j.re        B1[i][2j] = L_ij.re    B2[i][2j] =  L_ij.im
//     A[r][2j+1] = -v_r(nbr_k)_j.im        B1[i][2j+1] = L_ij.im  B2[i][2j+1] = -L_ij.re
//
//     (A B1^T)[r][i] = sum_j v.re L.re - v.im L.im = y_r,i.re
//     (A B2^T)[r][i] = sum_j v.re L.im + v.im L.re = y_r,i.im
//
// so D = A [B1; B2]^T (M = 128 rhs, N = 2N, K = 16 per instruction) accumulated over the 9 hops
// and all K steps in TMEM gives the complex result with no real-block expansion of the links.
// fp16 payloads are used as they are stored; the per-(site,k) link scale and the per-(site,rhs)
// vector scales enter as ratios <= 1 to their maxima (one HMUL2 per word) and are restored in
// the epilogue, which re-quantises every (site, rhs) record (R12).
//
// Layout of a multi-RHS field: [site][rhs][fp16 record] (record = N half2 + scale + pad).
// One CTA per (site, block of 128 rhs): 8 warps build the operands of hop k+1 in shared memory
// (core-matrix, no-swizzle K-major layout) while the tensor core runs hop k; one thread issues
// the MMAs and commits them to an mbarrier; warps 0-3 drain TMEM (tcgen05.ld) in the epilogue.
#include <cuda_fp16.h>
#include <cstdint>

#include "cd_internal.h"
#include "device_common.cuh"

namespace cd {

template <int NV>
struct MrhsCfg {
    static constexpr int N = 2 * NV;           // complex rows of a link matrix
    static constexpr int MR = 128;             // rhs per CTA (MMA M)
    static constexpr int NB = 2 * N;           // MMA N: B1 rows then B2 rows
    static constexpr int KCH = N / 4;          // 16-B K chunks per hop (8 halves = 4 complex)
    static constexpr int KSTEPS = KCH / 2;     // MMA K = 16 halves = 2 chunks
    static constexpr int LBO_A = (MR / 8) * 128;
    static constexpr int LBO_B = (NB / 8) * 128;
    static constexpr int A_BYTES = KCH * LBO_A;
    static constexpr int B_BYTES = KCH * LBO_B;
    static constexpr int OP = A_BYTES + B_BYTES;            // operand buffer (one hop)
    static constexpr int VREC = 4 * N + 16;                 // fp16 vector record
    static constexpr int MREC = 4 * N * N + 16;             // fp16 matrix record
    static constexpr int RAW_A = MR * VREC;                 // 128 neighbour records (contiguous)
    static constexpr int RAW = RAW_A;                       // raw stage: the records (links go via registers)
    static constexpr int HDR = 1024;                        // mbarriers, scales
    static constexpr int NRAW = 2;                          // raw prefetch depth (hops ahead)
    static constexpr int SMEM = HDR + OP + NRAW * RAW;      // 95 KB (N = 48): two CTAs per SM
    static constexpr int BCH = N * KCH;                     // 16-B chunks of one link matrix
    static constexpr int BPT = (BCH + 255) / 256;           // per thread
    static constexpr int APT = MR * KCH / 256;              // A chunks per thread
    static constexpr int THREADS = 256;
    static constexpr int TMEM_COLS = NB <= 128 ? 128 : 256;
    static_assert(NB % 16 == 0 && NB <= 256, "MMA N");
};

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    // SWIZZLE_NONE K-major canonical layout; version 1 (Blackwell); 16-byte units.
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

template <int M, int N>
__device__ __forceinline__ uint32_t idesc_f16_f32()
{
    // c_format F32 (bit 4), a/b format F16 (0), K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t half2_bits(float x)
{
    __half2 h = __float2half2_rn(x);
    return *reinterpret_cast<uint32_t *>(&h);
}
template <int NC>
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float *v)
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = __uint_as_float(r[q]);
}

// Hop order: X first (k = 8: this site's own records give the per-rhs reference scales), then 0..7.
__device__ __forceinline__ int mk_hop(int i) { return i == 0 ? 8 : i - 1; }

template <int NV>
__global__ void __launch_bounds__(MrhsCfg<NV>::THREADS, 2)
    dslash_mrhs(const unsigned char *__restrict__ links, const unsigned char *__restrict__ in, unsigned char *out,
                KGeom g, int nrhs, int dagger)
{
    using C = MrhsCfg<NV>;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *raw_full = reinterpret_cast<uint64_t *>(smem);         // [NRAW]
    uint64_t *mma_done = raw_full + 4;                               // [1]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + 64);
    float *inv_sr = reinterpret_cast<float *>(smem + 128);           // [128] 1 / s_v(x, r)
    float *ssl = reinterpret_cast<float *>(smem + 640);              // [1]   s_L(x, 8)
    unsigned char *op = smem + C::HDR;
    unsigned char *As = op, *Bs = op + C::A_BYTES;
    unsigned char *raw = op + C::OP;

    const int site = blockIdx.x;
    const int rb = blockIdx.y;   // block of 128 rhs
    const int tid = threadIdx.x, warp = tid >> 5;
    int x[4];
    decode(g, site, x);
    const unsigned char *lsite = links + (size_t)site * 9 * C::MREC;
    const size_t rhs0 = (size_t)rb * C::MR;

    if (warp == 0) {   // TMEM accumulator: 128 lanes x NB fp32 columns
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(tmem_slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // the 128 contiguous neighbour records of hop i -> ring slot i % NRAW (one bulk copy)
    auto issue_raw = [&](int i) {
        const int k = mk_hop(i);
        uint64_t *bar = &raw_full[i % C::NRAW];
        unsigned char *dst = raw + (i % C::NRAW) * C::RAW;
        mbar_arrive_expect_tx(bar, C::RAW_A);
        bulk_g2s(dst, in + ((size_t)neighbour(g, x, site, k) * nrhs + rhs0) * C::VREC, C::RAW_A, bar);
    };
    // link matrix of hop i -> registers (prefetched one hop ahead)
    uint4 bv[C::BPT];
    float bsc;
    auto load_b = [&](int i) {
        const unsigned char *mk = lsite + (size_t)mk_hop(i) * C::MREC;
#pragma unroll
        for (int u = 0; u < C::BPT; u++) {
            const int e = tid + u * C::THREADS;
            bv[u] = e < C::BCH ? ld_stream(mk + (size_t)e * 16) : make_uint4(0, 0, 0, 0);
        }
        bsc = ld_nc_f32(mk + 4 * C::N * C::N);
    };
    load_b(0);
    if (tid == 0) {
        for (int j = 0; j < C::NRAW; j++) mbar_init(&raw_full[j], 1);
        mbar_init(mma_done, 1);
        fence_mbar_init();
        for (int j = 0; j < C::NRAW; j++) issue_raw(j);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_f16_f32<C::MR, C::NB>();

    for (int i = 0; i < 9; i++) {
        const int k = mk_hop(i);
        const unsigned char *rs = raw + (i % C::NRAW) * C::RAW;
        mbar_wait(&raw_full[i % C::NRAW], (i / C::NRAW) & 1);
        if (i == 0) {   // reference scales: this site's own records (k = 8) and its X scale
            if (tid < C::MR) {
                const float s = *reinterpret_cast<const float *>(rs + tid * C::VREC + 4 * C::N);
                inv_sr[tid] = s > 0.0f ? __frcp_rn(s) : 0.0f;
            }
            if (tid == 0) ssl[0] = bsc;
            __syncthreads();
        }
        // the operand buffer is free once the MMAs of the previous hop completed
        if (i > 0) mbar_wait(mma_done, (i - 1) & 1);
        // ---- B1 / B2 rows (scaled by s_L(k)/s_L(8)) into the core-matrix layout
        {
            const float s8 = ssl[0];
            const uint32_t lr = half2_bits(s8 > 0.0f ? bsc * __frcp_rn(s8) : 0.0f);
#pragma unroll
            for (int u = 0; u < C::BPT; u++) {
                const int e = tid + u * C::THREADS;
                if (e >= C::BCH) continue;
                const int ii = e / C::KCH, c = e - ii * C::KCH;
                const uint32_t *w = &bv[u].x;
                uint4 b1, b2;
                uint32_t *o1 = &b1.x, *o2 = &b2.x;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const uint32_t sv = hmul2_u32(w[q], lr);                         // (re, im)
                    o1[q] = sv;
                    o2[q] = __byte_perm(sv, 0, 0x1032) ^ 0x80000000u;                // (im, -re)
                }
                *reinterpret_cast<uint4 *>(Bs + c * C::LBO_B + (ii >> 3) * 128 + (ii & 7) * 16) = b1;
                const int i2 = ii + C::N;
                *reinterpret_cast<uint4 *>(Bs + c * C::LBO_B + (i2 >> 3) * 128 + (i2 & 7) * 16) = b2;
            }
        }
        if (i + 1 < 9) load_b(i + 1);   // next hop's link matrix: in flight during this hop
        // ---- A rows: (re, -im) of the neighbour records scaled by s_v(nbr, r)/s_v(x, r); tau3 (dagger)
        // thread t: row r = t % 128, chunks c = t / 128 + 2u (all loads issued before use)
        {
            const int r = tid & (C::MR - 1), h = tid >> 7;
            const unsigned char *rec = rs + r * C::VREC;
            const uint32_t ratio = half2_bits(*reinterpret_cast<const float *>(rec + 4 * C::N) * inv_sr[r]);
            uint4 w4[C::APT];
#pragma unroll
            for (int u = 0; u < C::APT; u++) w4[u] = *reinterpret_cast<const uint4 *>(rec + (h + 2 * u) * 16);
#pragma unroll
            for (int u = 0; u < C::APT; u++) {
                const int c = h + 2 * u;
                const bool flip = dagger && (c * 4 >= NV);   // components j >= Nvec (4 complex per chunk)
                const uint32_t m = 0x80000000u ^ (flip ? 0x80008000u : 0u);
                const uint32_t *w = &w4[u].x;
                uint4 av;
                uint32_t *o = &av.x;
#pragma unroll
                for (int q = 0; q < 4; q++) o[q] = hmul2_u32(w[q] ^ m, ratio);
                *reinterpret_cast<uint4 *>(As + c * C::LBO_A + (r >> 3) * 128 + (r & 7) * 16) = av;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            if (i + C::NRAW < 9) issue_raw(i + C::NRAW);   // raw slot i % NRAW fully consumed
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(As);
            const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(Bs);
#pragma unroll
            for (int s = 0; s < C::KSTEPS; s++) {
                const uint64_t da = smem_desc(a0 + 2 * s * C::LBO_A, C::LBO_A, 128);
                const uint64_t db = smem_desc(b0 + 2 * s * C::LBO_B, C::LBO_B, 128);
                const uint32_t acc = (i > 0 || s > 0) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(mma_done))
                         : "memory");
        }
    }
    mbar_wait(mma_done, 8 & 1);   // the 9th commit: every MMA of this site is done
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- epilogue: warps 0-3, thread t <-> TMEM lane t <-> rhs t; two passes over TMEM (max, store)
    if (tid < C::MR) {
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
        const float scale = ssl[0] * (inv_sr[tid] > 0.0f ? __frcp_rn(inv_sr[tid]) : 0.0f);
        float mx = 0.0f;
#pragma unroll 1
        for (int cc = 0; cc < C::NB / 16; cc++) {
            float v[16];
            tmem_ld16<16>(lane_base + cc * 16, v);
#pragma unroll
            for (int q = 0; q < 16; q++) mx = fmaxf(mx, fabsf(v[q] * scale));
        }
        unsigned char *rec = out + ((size_t)site * nrhs + rhs0 + tid) * C::VREC;
#pragma unroll 1
        for (int cc = 0; cc < C::N / 16; cc++) {
            float re[16], im[16];
            tmem_ld16<16>(lane_base + cc * 16, re);
            tmem_ld16<16>(lane_base + C::N + cc * 16, im);
#pragma unroll
            for (int q4 = 0; q4 < 4; q4++) {
                uint4 o;
                uint32_t *ow = &o.x;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int i = cc * 16 + q4 * 4 + q;
                    const float sg = (dagger && i >= NV) ? -scale : scale;
                    const float yr = re[q4 * 4 + q] * sg, yi = im[q4 * 4 + q] * sg;
                    __half2 h = mx > 0.0f ? __halves2half2(__float2half_rn(__fdiv_rn(yr, mx)),
                                                           __float2half_rn(__fdiv_rn(yi, mx)))
                                          : __halves2half2(__float2half_rn(0.0f), __float2half_rn(0.0f));
                    ow[q] = *reinterpret_cast<uint32_t *>(&h);
                }
                *reinterpret_cast<uint4 *>(rec + (cc * 16 + q4 * 4) * 4) = o;
            }
        }
        *reinterpret_cast<float4 *>(rec + 4 * C::N) = make_float4(mx, 0.f, 0.f, 0.f);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

template <int NV>
static cudaError_t launch_mrhs_t(const void *links, const void *in, void *out, const KGeom &g, int nrhs, int dagger,
                                 cudaStream_t s)
{
    using C = MrhsCfg<NV>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(dslash_mrhs<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    count_launch();
    dslash_mrhs<NV><<<dim3((unsigned)g.V, (unsigned)(nrhs / C::MR)), C::THREADS, C::SMEM, s>>>(
        static_cast<const unsigned char *>(links), static_cast<const unsigned char *>(in),
        static_cast<unsigned char *>(out), g, nrhs, dagger);
    return cudaGetLastError();
}

cudaError_t launch_mrhs(int nvec, const void *links, const void *in, void *out, const KGeom &g, int nrhs, int dagger,
                        cudaStream_t s)
{
    if (nrhs % 128) return cudaErrorInvalidValue;
    return nvec == 24 ? launch_mrhs_t<24>(links, in, out, g, nrhs, dagger, s)
                      : launch_mrhs_t<32>(links, in, out, g, nrhs, dagger, s);
}

}  // namespace cd
