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
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int THREADS = 256;
    static constexpr int VREC = 4 * N + 16;    // fp16 vector record
    static constexpr int MREC = 4 * N * N + 16;
    static constexpr int SMEM = 2 * STAGE + 256;
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

template <int NV>
__global__ void __launch_bounds__(MrhsCfg<NV>::THREADS, 1)
    dslash_mrhs(const unsigned char *__restrict__ links, const unsigned char *__restrict__ in, unsigned char *out,
                KGeom g, int nrhs, int dagger)
{
    using C = MrhsCfg<NV>;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *stage_base = smem;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + 2 * C::STAGE);       // [0], [1]: stage MMA done
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + 2 * C::STAGE + 64);
    float *s_ratio_l = reinterpret_cast<float *>(smem + 2 * C::STAGE + 128);  // 9 link-scale ratios

    const int site = blockIdx.x;
    const int rb = blockIdx.y;   // block of 128 rhs
    const int tid = threadIdx.x, warp = tid >> 5;
    int x[4];
    decode(g, site, x);

    if (warp == 0) {   // TMEM accumulator: 128 lanes x NB fp32 columns
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(tmem_slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    // scales: S_L = max_k s_L(k); S_r = max_k s_v(nbr_k, r) for this thread's rhs r (tid < 128)
    const unsigned char *lsite = links + (size_t)site * 9 * C::MREC;
    float sl[9];
    float SL = 0.0f;
#pragma unroll
    for (int k = 0; k < 9; k++) {
        sl[k] = ld_nc_f32(lsite + (size_t)k * C::MREC + 4 * C::N * C::N);
        SL = fmaxf(SL, sl[k]);
    }
    int nb[9];
#pragma unroll
    for (int k = 0; k < 9; k++) nb[k] = neighbour(g, x, site, k);
    float Sr = 0.0f;
    if (tid < C::MR) {
        const size_t r = (size_t)rb * C::MR + tid;
#pragma unroll
        for (int k = 0; k < 9; k++)
            Sr = fmaxf(Sr, ld_nc_f32(in + ((size_t)nb[k] * nrhs + r) * C::VREC + 4 * C::N));
    }
    __shared__ float s_Sr[C::MR];
    if (tid < C::MR) s_Sr[tid] = Sr;
    if (tid < 9) s_ratio_l[tid] = SL > 0.0f ? sl[tid] / SL : 0.0f;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_f16_f32<C::MR, C::NB>();

    for (int k = 0; k < 9; k++) {
        const int st = k & 1;
        unsigned char *As = stage_base + st * C::STAGE;
        unsigned char *Bs = As + C::A_BYTES;
        // ---- load this hop's operands into registers (before waiting for the stage to free)
        const unsigned char *mk = lsite + (size_t)k * C::MREC;
        const uint32_t lr = half2_bits(s_ratio_l[k]);
        constexpr int BCH = C::N * C::KCH;                       // B1 chunks (rows x K-chunks)
        constexpr int BPT = (BCH + C::THREADS - 1) / C::THREADS;
        uint4 bv[BPT];
#pragma unroll
        for (int u = 0; u < BPT; u++) {
            const int e = tid + u * C::THREADS;
            bv[u] = e < BCH ? ld_stream(mk + (size_t)e * 16) : make_uint4(0, 0, 0, 0);   // row-major chunks
        }
        constexpr int ACH = C::MR * C::KCH;
        constexpr int APT = ACH / C::THREADS;
        uint4 av[APT];
        const unsigned char *vk = in + ((size_t)nb[k] * nrhs + (size_t)rb * C::MR) * C::VREC;
#pragma unroll
        for (int u = 0; u < APT; u++) {
            const int e = tid + u * C::THREADS;
            const int r = e / C::KCH, c = e - r * C::KCH;
            av[u] = ld_nc(vk + (size_t)r * C::VREC + c * 16);
        }
        // ---- the stage was last used by hop k-2: wait for its MMAs
        if (k >= 2) mbar_wait(&mbar[st], ((k - 2) >> 1) & 1);
        // ---- B1 / B2 rows (scaled by s_L(k)/S_L) into the core-matrix layout
#pragma unroll
        for (int u = 0; u < BPT; u++) {
            const int e = tid + u * C::THREADS;
            if (e >= BCH) continue;
            const int i = e / C::KCH, c = e - i * C::KCH;
            uint4 b1, b2;
            const uint32_t *w = &bv[u].x;
            uint32_t *o1 = &b1.x, *o2 = &b2.x;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t s = hmul2_u32(w[q], lr);                          // (re, im)
                o1[q] = s;
                o2[q] = __byte_perm(s, 0, 0x1032) ^ 0x80000000u;                  // (im, -re)
            }
            *reinterpret_cast<uint4 *>(Bs + c * C::LBO_B + (i >> 3) * 128 + (i & 7) * 16) = b1;
            const int i2 = i + C::N;
            *reinterpret_cast<uint4 *>(Bs + c * C::LBO_B + (i2 >> 3) * 128 + (i2 & 7) * 16) = b2;
        }
        // ---- A rows: (re, -im) of the neighbour vectors, scaled by s_v/S_r, tau3 for the dagger
#pragma unroll
        for (int u = 0; u < APT; u++) {
            const int e = tid + u * C::THREADS;
            const int r = e / C::KCH, c = e - r * C::KCH;
            const float sv = ld_nc_f32(vk + (size_t)r * C::VREC + 4 * C::N);
            const float S = s_Sr[r];
            const uint32_t ratio = half2_bits(S > 0.0f ? sv / S : 0.0f);
            const bool flip = dagger && (c * 4 >= NV);   // components j >= Nvec (4 complex per chunk)
            const uint32_t m = 0x80000000u ^ (flip ? 0x80008000u : 0u);
            uint4 a;
            const uint32_t *w = &av[u].x;
            uint32_t *o = &a.x;
#pragma unroll
            for (int q = 0; q < 4; q++) o[q] = hmul2_u32(w[q] ^ m, ratio);
            *reinterpret_cast<uint4 *>(As + c * C::LBO_A + (r >> 3) * 128 + (r & 7) * 16) = a;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(As);
            const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(Bs);
#pragma unroll
            for (int s = 0; s < C::KSTEPS; s++) {
                const uint64_t da = smem_desc(a0 + 2 * s * C::LBO_A, C::LBO_A, 128);
                const uint64_t db = smem_desc(b0 + 2 * s * C::LBO_B, C::LBO_B, 128);
                const uint32_t acc = (k > 0 || s > 0) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&mbar[st]))
                         : "memory");
        }
    }
    // all MMAs done: hop 8 used stage 0 (its 5th use: phase parity 0)
    mbar_wait(&mbar[0], 0);
    mbar_wait(&mbar[1], 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- epilogue: warps 0-3, thread t <-> TMEM lane t <-> rhs t
    if (tid < C::MR) {
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
        float yv[C::NB];
#pragma unroll
        for (int cc = 0; cc < C::NB / 16; cc++) {
            uint32_t r[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(lane_base + cc * 16));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int q = 0; q < 16; q++) yv[cc * 16 + q] = __uint_as_float(r[q]);
        }
        const float scale = s_Sr[tid] * SL;
        float mx = 0.0f;
#pragma unroll
        for (int i = 0; i < C::NB; i++) {
            const float sg = (dagger && (i % C::N) >= NV) ? -1.0f : 1.0f;
            yv[i] *= scale * sg;
            mx = fmaxf(mx, fabsf(yv[i]));
        }
        unsigned char *rec = out + ((size_t)site * nrhs + (size_t)rb * C::MR + tid) * C::VREC;
#pragma unroll
        for (int i = 0; i < C::N; i += 4) {
            uint4 o;
            uint32_t *ow = &o.x;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                __half2 h = mx > 0.0f ? __halves2half2(__float2half_rn(__fdiv_rn(yv[i + q], mx)),
                                                       __float2half_rn(__fdiv_rn(yv[C::N + i + q], mx)))
                                      : __halves2half2(__float2half_rn(0.0f), __float2half_rn(0.0f));
                ow[q] = *reinterpret_cast<uint32_t *>(&h);
            }
            *reinterpret_cast<uint4 *>(rec + i * 4) = o;
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
