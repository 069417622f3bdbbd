// mrhs.cu -- multi right-hand-side coarse Dslash on the 5th-generation tensor cores (tcgen05).
//
// SURVEY NEXT-1 (the paper's "multi-right-hand-side MG", §9): with n_rhs vectors
// the per-site work becomes a small GEMM, so tensor cores finally apply.  For one site x and
// one hop k, with A = the 128 right-hand sides' neighbour vectors v_r(nbr_k) as stored (row r =
// rhs, K index = 2j + {re,im}) and B built from the stored fp16 link matrix L_k(x) (row i =
// output colour-spin):
//
//     A[r][2j] = v.re   A[r][2j+1] = v.im      B1[i][2j] = L.re   B1[i][2j+1] = -L.im
//                                              B2[i][2j] = L.im   B2[i][2j+1] =  L.re
//     (A B1^T)[r][i] = y_r,i.re                (A B2^T)[r][i] = y_r,i.im
//
// so D = sum_k ratio_k A_k [B1_k; B2_k]^T (M = 128 rhs, N = 2N, K = 16 per instruction) in TMEM
// is the complex result with no real-block expansion of the links and NO transformation of A.
//
// Tensor-core field layout (R22): an fp16 multi-RHS field is stored as blocks of 128
// right-hand sides per site, [site][rhs block][K chunk c][rhs r][16 B] + one fp32 scale per
// (site, block): one 1-D bulk copy of a neighbour block lands in shared memory already in the
// UMMA SWIZZLE_NONE K-major canonical layout (core matrix = 8 rhs x 16 B, LBO = 2048 B between K
// chunks, SBO = 128 B between 8-row groups).  With one scale per block, every scale of hop k is a
// scalar: ratio_k = s_L(x,k) s_v(nbr_k) / s_ref, s_ref = max_k of the same products, folded into
// B (ratio <= 1: no fp16 overflow), restored in the epilogue, which re-quantises the block.
//
// Persistent warp-specialised kernel, one CTA per SM (two for Nvec 24: CPS = 2, a complete pipeline
// each in half the SM), items = (site, rhs block):
//   warp 0     producer: per hop one bulk copy of the neighbour block (A) + one of the link record
//              into an S-stage ring (mbarrier full/empty);
//   warp 1     MMA issuer (one thread): tcgen05.mma kind::f16 into a double-buffered TMEM
//              accumulator; tcgen05.commit releases ring stages, B slots and accumulators;
//   warps 2-5  B builders: raw link record -> B1/B2 rows (x ratio, dagger signs) in a
//              double-buffered B slot;
//   warps 6-9  epilogue: tcgen05.ld of the previous item's accumulator (the MMA already runs the
//              next item), s_ref / dagger / re-quantisation, coalesced 16-B stores.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "cd_internal.h"
#include "device_common.cuh"

namespace cd {

template <int NV, int NBS_ = (NV == 24 ? 3 : 2), int CPS_ = 1>
struct MrhsCfg {
    static constexpr int CPS = CPS_;           // CTAs per SM (2: two independent pipelines per SM)
    static constexpr int N = 2 * NV;           // complex rows of a link matrix
    static constexpr int MR = 128;             // rhs per block (MMA M)
    static constexpr int NB = 2 * N;           // MMA N: B1 rows then B2 rows
    static constexpr int KCH = N / 4;          // 16-B K chunks per hop (8 halves = 4 complex)
    static constexpr int KSTEPS = KCH / 2;     // MMA K = 16 halves = 2 chunks
    static constexpr int LBO_A = MR * 16;      // 2048: one K chunk of all 128 rhs
    static constexpr int LBO_B = NB * 16;
    static constexpr int A_BYTES = KCH * LBO_A;            // block payload
    static constexpr int BLK = A_BYTES + 16;               // + scale (16-B padded)
    static constexpr int B_BYTES = KCH * LBO_B;
    static constexpr int MREC = 4 * N * N + 16;            // fp16 matrix record
    static constexpr int STAGE = (BLK + MREC + 127) / 128 * 128;
    static constexpr int HDR = 1024;
    static constexpr int SMEM_MAX = CPS == 1 ? 232448 : 115712;      // per CTA (2 CTAs: 228 KB - 2 x 1 KB reserved)
    static constexpr int NBS = NBS_;                                   // B slots (builders run ahead)
    static constexpr int S = (SMEM_MAX - HDR - NBS * B_BYTES) / STAGE;  // ring stages
    static constexpr int SMEM = HDR + NBS * B_BYTES + S * STAGE;
    static constexpr int BCH = N * KCH;                     // 16-B chunks of one link matrix
    static constexpr int NBW = 6;                           // builder warps
    static constexpr int NBT = 32 * NBW;
    static constexpr int EPI0 = 2 + NBW;                    // first epilogue warp
    static constexpr int THREADS = 32 * (EPI0 + 4);
    static constexpr int TMEM_COLS = 2 * NB <= 256 ? 256 : 512;
    static_assert(S >= 2 && S <= 6, "ring size (barrier slots)");
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
// 16 consecutive TMEM columns of this warp's 32 lanes (no wait: the caller waits once for all,
// then passes the registers through reg_fence16 so no use is scheduled above the wait)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t addr, uint32_t *r)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
__device__ __forceinline__ void reg_fence16(uint32_t *r)
{
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]));
}


// Item -> (site, rhs block), lexicographic: the ~148 items in flight are consecutive sites, which
// share most of their neighbour lines in L2 (a 4-D Morton order was measured 7 % slower).
__device__ __forceinline__ int item_site(int64_t it, int nrb, int &rb, const int *sites)
{
    const int z = (int)(it / nrb);
    rb = (int)(it - (int64_t)z * nrb);
    return sites ? __ldg(sites + z) : z;
}

// The A block of hop k: the neighbour's block in this rank's field, or -- for a hop that leaves
// the rank (multi-rank) -- its copy in the halo receive buffer: a +mu hop reads block B (sent by
// the +mu neighbour from its x_mu = 0 face), a -mu hop block A (R13 order, per rhs block).
// hl.off[mu][blk] without dynamic indexing of a kernel parameter (which would force a local copy)
__device__ __forceinline__ int64_t halo_off(const MrhsHalo &hl, int mu, int blk)
{
    const int64_t a0 = blk ? hl.off[0][1] : hl.off[0][0], a1 = blk ? hl.off[1][1] : hl.off[1][0];
    const int64_t a2 = blk ? hl.off[2][1] : hl.off[2][0], a3 = blk ? hl.off[3][1] : hl.off[3][0];
    return mu == 0 ? a0 : (mu == 1 ? a1 : (mu == 2 ? a2 : a3));
}

template <int BLK>
__device__ __forceinline__ const unsigned char *nbr_block(const KGeom &g, const MrhsHalo &hl, const unsigned char *in,
                                                          const int x[4], int site, int k, int nrb, int rb)
{
    if (hl.recv != nullptr && remote_hop(g, x, k)) {
        const int mu = k >> 1;
        const int blk = (k & 1) ? 0 : 1;
        // face index: lexicographic over the other three dims (no dynamic register indexing)
        const int f = mu == 0 ? (x[3] * g.L[2] + x[2]) * g.L[1] + x[1]
                    : mu == 1 ? (x[3] * g.L[2] + x[2]) * g.L[0] + x[0]
                    : mu == 2 ? (x[3] * g.L[1] + x[1]) * g.L[0] + x[0]
                              : (x[2] * g.L[1] + x[1]) * g.L[0] + x[0];
        return static_cast<const unsigned char *>(hl.recv) + halo_off(hl, mu, blk) + ((size_t)f * nrb + rb) * BLK;
    }
    return in + ((size_t)neighbour(g, x, site, k) * nrb + rb) * BLK;
}

__device__ __forceinline__ void st_evict_first(void *p, uint4 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
}

// hop products s_L(x,k) * s_v(nbr_k, block) and their max (identical in builders and epilogue)
template <int NV>
__device__ __forceinline__ float hop_scale(const unsigned char *links, const unsigned char *in, const KGeom &g,
                                           const MrhsHalo &hl, const int x[4], int site, int k, int nrb, int rb)
{
    using C = MrhsCfg<NV, 2>;
    const float sl = ld_nc_f32(links + ((size_t)site * 9 + k) * C::MREC + 4 * C::N * C::N);
    const float sv = ld_nc_f32(nbr_block<C::BLK>(g, hl, in, x, site, k, nrb, rb) + C::A_BYTES);
    return sl * sv;
}

template <int NV, int NBS, int CPS>
__global__ void __launch_bounds__(MrhsCfg<NV, NBS, CPS>::THREADS, CPS)
    dslash_mrhs(const unsigned char *__restrict__ links, const unsigned char *__restrict__ in, unsigned char *out,
                KGeom g, int nrb, int dagger, const int *sites, int nsites, MrhsHalo hl, long long *trace, int pf,
                int smax, int exp)
{
    using C = MrhsCfg<NV, NBS, CPS>;
    // optional diagnostic trace of CTA 0 (CD_MRHS_TRACE): trace[ev * 512 + index] = clock64(), 12 events
    const bool tr = trace != nullptr && blockIdx.x == 0;
#define TR(ev, idx) \
    if (tr && (idx) < 512) trace[(ev) * 512 + (idx)] = clock64();
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);       // [S]
    uint64_t *empty = full + 16;                                 // [S]
    uint64_t *lempty = full + 52;                                // [S]
    uint64_t *lfull = full + 58;                                 // [S] link record landed (exp & 32)
    uint64_t *bfull = full + 32;                                 // [NBS]
    uint64_t *bempty = full + 40;                                // [NBS]
    uint64_t *accfull = full + 48;                               // [2]
    uint64_t *accempty = full + 50;                              // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + 512);
    float *red = reinterpret_cast<float *>(smem + 640);          // [4] epilogue max
    float *hs = reinterpret_cast<float *>(smem + 704);           // [2][9] builder hop scales
    float *es = reinterpret_cast<float *>(smem + 800);           // [9]    epilogue hop scales
    unsigned char *bbuf = smem + C::HDR;                         // [NBS][B_BYTES]
    unsigned char *ring = bbuf + C::NBS * C::B_BYTES;            // [S][STAGE]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t items = (int64_t)(sites ? nsites : g.V) * nrb;

    if (tid == 0) {
        for (int j = 0; j < C::S; j++) {
            mbar_init(&full[j], 1);
            mbar_init(&empty[j], 1);            // the MMA commit (A consumed by the tensor core)
            mbar_init(&lempty[j], (exp & 16) ? C::NBW : C::NBT);   // builder threads (or warps) done with the link
            mbar_init(&lfull[j], 1);
        }
        for (int j = 0; j < C::NBS; j++) {
            mbar_init(&bfull[j], C::NBW);
            mbar_init(&bempty[j], 1);
        }
        for (int j = 0; j < 2; j++) {
            mbar_init(&accfull[j], 1);
            mbar_init(&accempty[j], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(tmem_slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "n"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol_v = l2_policy_evict_last(), pol_l = l2_policy_evict_first();
            uint32_t h = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                int rb;
                const int site = item_site(it, nrb, rb, sites);
                int x[4];
                decode(g, site, x);
                // L2 prefetch of the next item's 9 link records (one contiguous run, read from DRAM
                // once per apply): the ring's link copies then see L2 rather than DRAM latency.
                // Nvec 32 (16 KB records): 147 -> 144 us at 6^3x12 x 128; Nvec 24: neutral to 1 %
                // slower, off.  Prefetching the neighbour blocks too was slower for both
                // (profiles/r02/mrhs_l2_prefetch_ab.txt).
                if (pf && it + gridDim.x < items) {
                    int rbp;
                    const int sp = item_site(it + gridDim.x, nrb, rbp, sites);
                    bulk_prefetch_l2(links + (size_t)sp * 9 * C::MREC, 9 * C::MREC);
                }
                for (int k = 0; k < 9; k++, h++) {
                    const int st = h % smax;
                    mbar_wait(&empty[st], ((h / smax) & 1) ^ 1);
                    mbar_wait(&lempty[st], ((h / smax) & 1) ^ 1);
                    unsigned char *dst = ring + st * C::STAGE;
                    TR(10, h)
                    // vectors are re-read by 9 sites (keep them in L2), links are read once
                    if (exp & 32) {
                        // link first, on its own barrier: the B build overlaps the neighbour block's flight
                        mbar_arrive_expect_tx(&lfull[st], C::MREC);
                        bulk_g2s_hint(dst + C::BLK, links + ((size_t)site * 9 + k) * C::MREC, C::MREC, &lfull[st],
                                      pol_l);
                        mbar_arrive_expect_tx(&full[st], C::BLK);
                        bulk_g2s_hint(dst, nbr_block<C::BLK>(g, hl, in, x, site, k, nrb, rb), C::BLK, &full[st],
                                      pol_v);
                    } else {
                    mbar_arrive_expect_tx(&full[st], ((exp & 8) ? 0 : C::BLK) + ((exp & 4) ? 0 : C::MREC));
                    if (!(exp & 8))
                        bulk_g2s_hint(dst, nbr_block<C::BLK>(g, hl, in, x, site, k, nrb, rb), C::BLK,
                                      &full[st], pol_v);
                    if (!(exp & 4))
                        bulk_g2s_hint(dst + C::BLK, links + ((size_t)site * 9 + k) * C::MREC, C::MREC, &full[st],
                                      pol_l);
                    }
                    TR(0, h)
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_f16_f32<C::MR, C::NB>();
            const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring);
            const uint32_t bb0 = (uint32_t)__cvta_generic_to_shared(bbuf);
            uint32_t h = 0, t = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x, t++) {
                const int acc = t & 1;
                mbar_wait(&accempty[acc], ((t >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + acc * C::NB;
                TR(9, t)
                for (int k = 0; k < 9; k++, h++) {
                    const int st = h % smax, bs = h % C::NBS;
                    // merged hand-offs (exp & 64): the builders publish B only once the neighbour block
                    // has landed too, so bfull alone gates the MMA
                    if (!(exp & 64)) mbar_wait(&full[st], (h / smax) & 1);
                    TR(1, h)
                    mbar_wait(&bfull[bs], (h / C::NBS) & 1);
                    TR(2, h)
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a0 = ring0 + st * C::STAGE, b0 = bb0 + bs * C::B_BYTES;
#pragma unroll
                    for (int s = 0; s < C::KSTEPS; s++) {
                        if (exp & 2) break;
                        const uint64_t da = smem_desc(a0 + 2 * s * C::LBO_A, C::LBO_A, 128);
                        const uint64_t db = smem_desc(b0 + 2 * s * C::LBO_B, C::LBO_B, 128);
                        const uint32_t accum = (k > 0 || s > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                            "l"(da), "l"(db), "r"(idesc), "r"(accum));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(&empty[st]))
                                 : "memory");
                    if (!(exp & 64))   // merged: the builders wait on the stage's empty barrier instead
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                         (uint32_t)__cvta_generic_to_shared(&bempty[bs]))
                                     : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(&accfull[acc]))
                             : "memory");
            }
        }
    } else if (warp < C::EPI0) {
        // ------------------------------------------------------------ B builders (NBW warps)
        const int bt = tid - 64;
        constexpr int UPT = (C::BCH + C::NBT - 1) / C::NBT;   // 16-B chunks per thread per hop
        uint32_t h = 0, t = 0;
        // hop scales of the NEXT item are loaded one item ahead (their latency hides behind 9 hops)
        float nsl = 0.0f, nsv = 0.0f;   // raw loads, multiplied only when consumed
        auto scale_of = [&](int64_t it) {
            int rb;
                const int site = item_site(it, nrb, rb, sites);
            int x[4];
            decode(g, site, x);
            nsl = ld_nc_f32(links + ((size_t)site * 9 + bt) * C::MREC + 4 * C::N * C::N);
            nsv = ld_nc_f32(nbr_block<C::BLK>(g, hl, in, x, site, bt, nrb, rb) + C::A_BYTES);
        };
        if (bt < 9 && (int64_t)blockIdx.x < items) scale_of(blockIdx.x);
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x, t++) {
            float *hsb = hs + (t & 1) * 9;
            if (bt < 9) {
                hsb[bt] = nsl * nsv;   // == hop_scale (same fp32 product as the epilogue)
                if (it + gridDim.x < items) scale_of(it + gridDim.x);
            }
            bar_named(1, C::NBT);
            float sref = 0.0f;
#pragma unroll
            for (int k = 0; k < 9; k++) sref = fmaxf(sref, hsb[k]);
            const float isref = sref > 0.0f ? __frcp_rn(sref) : 0.0f;
            for (int k = 0; k < 9; k++, h++) {
                const int st = h % smax, bs = h % C::NBS;
                const uint32_t ratio = half2_bits(hsb[k] * isref);
                if (exp & 64) {
                    // B slot bs was last read by hop h - NBS, whose commit completes phase (h - NBS) / S of
                    // that hop's stage barrier (it cannot be a later phase: hop h + S - NBS needs this B)
                    if (h >= (uint32_t)C::NBS) {
                        const uint32_t hp = h - C::NBS;
                        mbar_wait(&empty[hp % smax], (hp / smax) & 1);
                    }
                } else {
                    mbar_wait(&bempty[bs], ((h / C::NBS) & 1) ^ 1);
                }
                if (bt == 0) TR(3, h)
                mbar_wait((exp & 32) ? &lfull[st] : &full[st], (h / smax) & 1);
                if (exp & 1) {
                    if (!(exp & 16) || lane == 0) mbar_arrive(&lempty[st]);
                    if (exp & 64) mbar_wait(&full[st], (h / smax) & 1);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bfull[bs]);
                    continue;
                }
                if (bt == 0) TR(4, h)
                const unsigned char *lraw = ring + st * C::STAGE + C::BLK;
                unsigned char *Bs = bbuf + bs * C::B_BYTES;
                // bank-conflict-free for both sides: the 8 threads of a 128-bit access phase take 8
                // consecutive rows (distinct 16-B slots of a B core matrix) and chunks c0 + t/2
                // (the raw row stride of 12 or 16 chunks would otherwise alias)
                uint4 w[UPT];
                int ii[UPT], cc[UPT];
#pragma unroll
                for (int u = 0; u < UPT; u++) {
                    const int e = bt + u * C::NBT;
                    const int t8 = e & 7, grp = e >> 3;
                    const int rbk = grp % (C::N / 8), cb = grp / (C::N / 8);
                    ii[u] = rbk * 8 + t8;
                    const int c = cb + (t8 >> 1);
                    cc[u] = c >= C::KCH ? c - C::KCH : c;
                    if (e < C::BCH) w[u] = *reinterpret_cast<const uint4 *>(lraw + ((size_t)ii[u] * C::KCH + cc[u]) * 16);
                }
                if (exp & 16) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&lempty[st]);   // the warp is done with the stage's link record
                } else {
                    mbar_arrive(&lempty[st]);   // this thread is done with the stage's link record
                }
#pragma unroll
                for (int u = 0; u < UPT; u++) {
                    if (bt + u * C::NBT >= C::BCH) break;
                    const int c = cc[u];
                    const uint32_t flip = (dagger && c * 4 >= NV) ? 0x80008000u : 0u;   // tau3 on the input
                    uint4 b1, b2;
                    uint32_t *wi = &w[u].x, *o1 = &b1.x, *o2 = &b2.x;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t v = hmul2_u32(wi[q] ^ flip, ratio);             // (re, im)
                        o1[q] = v ^ 0x80000000u;                                       // (re, -im)
                        o2[q] = __byte_perm(v, 0, 0x1032);                             // (im, re)
                    }
                    *reinterpret_cast<uint4 *>(Bs + c * C::LBO_B + (ii[u] >> 3) * 128 + (ii[u] & 7) * 16) = b1;
                    const int i2 = ii[u] + C::N;
                    *reinterpret_cast<uint4 *>(Bs + c * C::LBO_B + (i2 >> 3) * 128 + (i2 & 7) * 16) = b2;
                }
                if (exp & 64) mbar_wait(&full[st], (h / smax) & 1);   // the neighbour block landed too
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&bfull[bs]);
                if (bt == 0) TR(5, h)
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (128 threads)
        const int et = tid - 32 * C::EPI0;
        const uint64_t pol_o = l2_policy_evict_first();   // outputs are not re-read by this apply
        const int r = 32 * (warp & 3) + lane;   // TMEM lane = rhs row (warp w reaches lanes 32(w%4)..)
        uint32_t t = 0;
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x, t++) {
            int rb;
                const int site = item_site(it, nrb, rb, sites);
            int x[4];
            decode(g, site, x);
            if (et < 9) es[et] = hop_scale<NV>(links, in, g, hl, x, site, et, nrb, rb);
            const int acc = t & 1;
            if (et == 0) TR(6, t)
            mbar_wait(&accfull[acc], (t >> 1) & 1);
            if (et == 0) TR(7, t)
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t base = tmem + acc * C::NB + ((uint32_t)(32 * (warp & 3)) << 16);
            if constexpr (C::CPS == 2) {
                // two CTAs per SM (<= 85 registers per thread): two passes over the accumulator in
                // tensor memory -- the block max, then re-quantise and store -- in chunks of columns
                bar_named(2, 128);                          // es[] visible
                float sref = 0.0f;
#pragma unroll
                for (int k = 0; k < 9; k++) sref = fmaxf(sref, es[k]);
                float m = 0.0f;
#pragma unroll 1
                for (int cc = 0; cc < C::NB / 16; cc++) {
                    uint32_t r16[16];
                    tmem_ld16_nowait(base + cc * 16, r16);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    reg_fence16(r16);
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int col = cc * 16 + i, row = col < C::N ? col : col - C::N;
                        m = fmaxf(m, fabsf(__uint_as_float(r16[i]) * ((dagger && row >= NV) ? -sref : sref)));
                    }
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                if (lane == 0) red[warp & 3] = m;
                bar_named(2, 128);
                m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
                unsigned char *blk = out + ((size_t)site * nrb + rb) * C::BLK;
                const float im = m > 0.0f ? __frcp_rn(m) : 0.0f;
#pragma unroll 1
                for (int c = 0; c < C::KCH; c++) {
                    uint32_t re4[4], im4[4];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(re4[0]), "=r"(re4[1]), "=r"(re4[2]), "=r"(re4[3]) : "r"(base + 4 * c));
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(im4[0]), "=r"(im4[1]), "=r"(im4[2]), "=r"(im4[3]) : "r"(base + C::N + 4 * c));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    uint4 o;
                    uint32_t *ow = &o.x;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const int row = 4 * c + q;
                        const float sg = (dagger && row >= NV) ? -sref : sref;
                        asm volatile("" : "+r"(re4[q]), "+r"(im4[q]));
                        __half2 hv = __floats2half2_rn(__uint_as_float(re4[q]) * sg * im, __uint_as_float(im4[q]) * sg * im);
                        ow[q] = *reinterpret_cast<uint32_t *>(&hv);
                    }
                    st_evict_first(blk + c * C::LBO_A + r * 16, o, pol_o);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&accempty[acc]);   // the MMA may reuse this accumulator
                if (et == 0) *reinterpret_cast<float4 *>(blk + C::A_BYTES) = make_float4(m, 0.f, 0.f, 0.f);
                bar_named(2, 128);   // red[] / es[] reuse by the next item
                continue;
            }
            uint32_t raw[C::NB];
#pragma unroll
            for (int cc = 0; cc < C::NB / 16; cc++) tmem_ld16_nowait(base + cc * 16, raw + cc * 16);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int cc = 0; cc < C::NB / 16; cc++) reg_fence16(raw + cc * 16);
            float v[C::NB];
#pragma unroll
            for (int i = 0; i < C::NB; i++) v[i] = __uint_as_float(raw[i]);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[acc]);   // the MMA may reuse this accumulator
            bar_named(2, 128);                              // es[] visible
            float sref = 0.0f;
#pragma unroll
            for (int k = 0; k < 9; k++) sref = fmaxf(sref, es[k]);
            float m = 0.0f;
#pragma unroll
            for (int i = 0; i < C::NB; i++) {
                const int row = i < C::N ? i : i - C::N;
                v[i] *= (dagger && row >= NV) ? -sref : sref;
                m = fmaxf(m, fabsf(v[i]));
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red[warp & 3] = m;
            bar_named(2, 128);
            m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
            unsigned char *blk = out + ((size_t)site * nrb + rb) * C::BLK;
            // re-quantisation by the reciprocal (R22: x * (1/s), one cvt.rn.f16x2 per pair)
            const float im = m > 0.0f ? __frcp_rn(m) : 0.0f;
#pragma unroll
            for (int c = 0; c < C::KCH; c++) {
                uint4 o;
                uint32_t *ow = &o.x;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int i = 4 * c + q;
                    __half2 hv = __floats2half2_rn(v[i] * im, v[C::N + i] * im);
                    ow[q] = *reinterpret_cast<uint32_t *>(&hv);
                }
                st_evict_first(blk + c * C::LBO_A + r * 16, o, pol_o);
            }
            if (et == 0) *reinterpret_cast<float4 *>(blk + C::A_BYTES) = make_float4(m, 0.f, 0.f, 0.f);
            if (et == 0) TR(8, t)
            bar_named(2, 128);   // red[] / es[] reuse by the next item
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

template <int NV, int NBS, int CPS = 1>
static cudaError_t launch_mrhs_t(const void *links, const void *in, void *out, const KGeom &g, int nrhs, int dagger,
                                 cudaStream_t s, int num_sms, const int *sites, int nsites, const MrhsHalo *halo)
{
    using C = MrhsCfg<NV, NBS, CPS>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(dslash_mrhs<NV, NBS, CPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int nrb = nrhs / C::MR;
    const int64_t items = (int64_t)(sites ? nsites : g.V) * nrb;
    if (items == 0) return cudaSuccess;
    MrhsHalo hl{};
    if (halo) hl = *halo;
    count_launch();
    const char *pfe = getenv("CD_MRHS_PF");   // A/B switch: 0 / 1 override the per-Nvec default
    const int pf = pfe ? atoi(pfe) : (NV == 32);
    // diagnostic knobs (timing experiments only; results are wrong with exp != 0): CD_MRHS_SMAX caps the
    // ring stages, CD_MRHS_EXP bit 0 = builders skip the B build, 1 = no MMA, 2 = no link copy, 3 = no A copy,
    // 4 = per-warp link release (no change), 5 = link on its own barrier (the default), 6 = merged hand-offs
    // (measured 4-11 % slower)
    const char *sme = getenv("CD_MRHS_SMAX"), *exe = getenv("CD_MRHS_EXP");
    const int smax = sme && atoi(sme) >= 2 && atoi(sme) < C::S ? atoi(sme) : C::S;
    // default 32: the link record on its own barrier, issued before the neighbour block (B build overlaps
    // the block's flight): 8^4 x 128 152 -> 149 us, 6^3x12 148 -> 143 us (profiles/r02/mrhs_release.txt)
    const int exp = exe ? atoi(exe) : 32;
    long long *trace = nullptr;
    const char *tf = getenv("CD_MRHS_TRACE");   // diagnostic only: per-event clock64 of CTA 0
    if (tf) {
        cudaMalloc(&trace, 12 * 512 * sizeof(long long));
        cudaMemsetAsync(trace, 0, 12 * 512 * sizeof(long long), s);
    }
    const int64_t gmax = (int64_t)CPS * num_sms;
    dslash_mrhs<NV, NBS, CPS><<<(unsigned)(items < gmax ? items : gmax), C::THREADS, C::SMEM, s>>>(
        static_cast<const unsigned char *>(links), static_cast<const unsigned char *>(in),
        static_cast<unsigned char *>(out), g, nrb, dagger, sites, nsites, hl, trace, pf, smax, exp);
    cudaError_t e = cudaGetLastError();
    if (tf) {
        long long h[12 * 512];
        cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        cudaFree(trace);
        if (FILE *f = fopen(tf, "wb")) {
            fwrite(h, sizeof(h), 1, f);
            fclose(f);
        }
    }
    return e;
}

// ===================================================================================== TS variant
// The same product with the roles swapped (round 2): the LINK is the MMA's A operand, built by the
// builder warps straight into tensor memory (tcgen05.st), and the stored neighbour block is the B
// operand (N = 128 rhs, K-major exactly as stored: same descriptor as the A of the kernel above):
//
//     D[m][r] = sum_K A_k[m][K] v_r(nbr_k)[K],   A_k row 2i = ratio_k (L_i.re, -L_i.im),
//                                                A_k row 2i+1 = ratio_k (L_i.im, L_i.re)
//
// so D lane 2i holds y_i.re and lane 2i+1 y_i.im for every rhs column (M = 128 lanes, 2N = 96 or
// 128 of them used; with Nvec 24 lanes 96-127 are never written and never read).  No B slots in
// shared memory: the ring gets one more stage (Nvec 24: 6, Nvec 32: 4) and a hop's link no longer
// crosses shared memory twice more (B build write + MMA read).  The epilogue re-quantises through a
// padded shared staging tile (pitch 2080 B per K chunk: conflict-free 32-bit stores) that leaves
// with one bulk store per K chunk.
template <int NV>
struct MrhsTsCfg {
    static constexpr int N = 2 * NV;
    static constexpr int MR = 128;                          // rhs per block (MMA N)
    static constexpr int KCH = N / 4;                       // 16-B K chunks per hop
    static constexpr int KSTEPS = KCH / 2;                  // MMA K = 16 halves
    static constexpr int LBO = MR * 16;                     // 2048
    static constexpr int A_BYTES = KCH * LBO;
    static constexpr int BLK = A_BYTES + 16;
    static constexpr int MREC = 4 * N * N + 16;
    static constexpr int STAGE = (BLK + MREC + 127) / 128 * 128;
    static constexpr int ACOLS = N;                         // 32-bit TMEM columns of one A slot (2N halves)
    static constexpr int NBS = NV == 24 ? 5 : 4;            // A slots in TMEM (the builders run ahead)
    static constexpr int PITCH = LBO + 32;                  // staging pitch per K chunk
    static constexpr int STG = KCH * PITCH;
    static constexpr int HDR = 1024;
    static constexpr int SMEM_MAX = 232448;
    static constexpr int S = (SMEM_MAX - HDR - STG) / STAGE;
    static constexpr int SMEM = HDR + STG + S * STAGE;
    static constexpr int NBT = 128;                         // builder threads (warps 2-5)
    static constexpr int THREADS = 320;                     // + epilogue warps 6-9
    static constexpr int DCOL = 0, ACOL = 2 * MR;           // TMEM: two accumulators, then A slots
    static_assert(S >= 2, "ring too small");
    static_assert(ACOL + NBS * ACOLS <= 512, "TMEM columns");
    static_assert(S <= 8 && NBS <= 8, "barrier slots");
};

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t *r)
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void *dst, const void *src_smem, uint32_t bytes, uint64_t pol)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"((uint32_t)__cvta_generic_to_shared(src_smem)), "r"(bytes), "l"(pol)
                 : "memory");
}

template <int NV>
__global__ void __launch_bounds__(MrhsTsCfg<NV>::THREADS, 1)
    dslash_mrhs_ts(const unsigned char *__restrict__ links, const unsigned char *__restrict__ in, unsigned char *out,
                   KGeom g, int nrb, int dagger, const int *sites, int nsites, MrhsHalo hl, int pf)
{
    using C = MrhsTsCfg<NV>;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);       // [S]
    uint64_t *empty = full + 16;                                 // [S]
    uint64_t *lempty = full + 32;                                // [S]
    uint64_t *bfull = full + 48;                                 // [NBS]
    uint64_t *bempty = full + 40;                                // [NBS]
    uint64_t *accfull = full + 56;                               // [2]
    uint64_t *accempty = full + 58;                              // [2]
    uint64_t *lfull = full + 24;                                 // [S] link record landed
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + 512);
    float *red = reinterpret_cast<float *>(smem + 640);          // [4] epilogue max
    float *hs = reinterpret_cast<float *>(smem + 704);           // [2][9] builder hop scales
    float *es = reinterpret_cast<float *>(smem + 800);           // [9]    epilogue hop scales
    unsigned char *stg = smem + C::HDR;                          // [KCH][PITCH] output staging
    unsigned char *ring = stg + C::STG;                          // [S][STAGE]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t items = (int64_t)(sites ? nsites : g.V) * nrb;

    if (tid == 0) {
        for (int j = 0; j < C::S; j++) {
            mbar_init(&full[j], 1);
            mbar_init(&empty[j], 1);            // the MMA commit (B = neighbour block consumed)
            mbar_init(&lempty[j], C::NBT);      // every builder thread (raw link record read)
            mbar_init(&lfull[j], 1);
        }
        for (int j = 0; j < C::NBS; j++) {
            mbar_init(&bfull[j], 4);            // one arrival per builder warp
            mbar_init(&bempty[j], 1);
        }
        for (int j = 0; j < 2; j++) {
            mbar_init(&accfull[j], 1);
            mbar_init(&accempty[j], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(tmem_slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer (as dslash_mrhs)
        if (lane == 0) {
            const uint64_t pol_v = l2_policy_evict_last(), pol_l = l2_policy_evict_first();
            uint32_t h = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                int rb;
                const int site = item_site(it, nrb, rb, sites);
                int x[4];
                decode(g, site, x);
                if (pf && it + gridDim.x < items) {
                    int rbp;
                    const int sp = item_site(it + gridDim.x, nrb, rbp, sites);
                    bulk_prefetch_l2(links + (size_t)sp * 9 * C::MREC, 9 * C::MREC);
                }
#pragma unroll 1
                for (int k = 0; k < 9; k++, h++) {
                    const int st = h % C::S;
                    mbar_wait(&empty[st], ((h / C::S) & 1) ^ 1);
                    mbar_wait(&lempty[st], ((h / C::S) & 1) ^ 1);
                    unsigned char *dst = ring + st * C::STAGE;
                    mbar_arrive_expect_tx(&lfull[st], C::MREC);
                    bulk_g2s_hint(dst + C::BLK, links + ((size_t)site * 9 + k) * C::MREC, C::MREC, &lfull[st], pol_l);
                    mbar_arrive_expect_tx(&full[st], C::BLK);
                    bulk_g2s_hint(dst, nbr_block<C::BLK>(g, hl, in, x, site, k, nrb, rb), C::BLK, &full[st], pol_v);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (A in TMEM, B in smem)
        if (lane == 0) {
            // F32 accumulate, F16 A/B, both K-major, N = 128 (>> 3 at bit 17), M = 128 (>> 4 at bit 24)
            const uint32_t idesc = (1u << 4) | ((uint32_t)(C::MR >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring);
            uint32_t h = 0, t = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x, t++) {
                const int acc = t & 1;
                mbar_wait(&accempty[acc], ((t >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + C::DCOL + acc * C::MR;
#pragma unroll 1
                for (int k = 0; k < 9; k++, h++) {
                    const int st = h % C::S, bs = h % C::NBS;
                    mbar_wait(&full[st], (h / C::S) & 1);
                    mbar_wait(&bfull[bs], (h / C::NBS) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t b0 = ring0 + st * C::STAGE, a0 = tmem + C::ACOL + bs * C::ACOLS;
#pragma unroll
                    for (int s = 0; s < C::KSTEPS; s++) {
                        const uint64_t db = smem_desc(b0 + 2 * s * C::LBO, C::LBO, 128);
                        const uint32_t accum = (k > 0 || s > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                            "r"(a0 + 8 * s), "l"(db), "r"(idesc), "r"(accum));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(&empty[st]))
                                 : "memory");
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(&bempty[bs]))
                                 : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(&accfull[acc]))
                             : "memory");
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------------------ A builders (warps 2-5)
        // warp w may only reach TMEM lanes 32 (w % 4) .. + 31: this thread owns lane (= A row) m
        const int bt = tid - 64, q = warp & 3, m = 32 * q + lane;
        const bool live = m < 2 * C::N;
        const int i = m >> 1, part = m & 1;
        const uint32_t lrow = (uint32_t)(32 * q) << 16;
        uint32_t h = 0, t = 0;
        float nsl = 0.0f, nsv = 0.0f;
        auto scale_of = [&](int64_t it) {
            int rb;
            const int site = item_site(it, nrb, rb, sites);
            int x[4];
            decode(g, site, x);
            nsl = ld_nc_f32(links + ((size_t)site * 9 + bt) * C::MREC + 4 * C::N * C::N);
            nsv = ld_nc_f32(nbr_block<C::BLK>(g, hl, in, x, site, bt, nrb, rb) + C::A_BYTES);
        };
        if (bt < 9 && (int64_t)blockIdx.x < items) scale_of(blockIdx.x);
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x, t++) {
            float *hsb = hs + (t & 1) * 9;
            if (bt < 9) {
                hsb[bt] = nsl * nsv;   // == hop_scale (same fp32 product as the epilogue)
                if (it + gridDim.x < items) scale_of(it + gridDim.x);
            }
            bar_named(1, C::NBT);
            float sref = 0.0f;
#pragma unroll
            for (int k = 0; k < 9; k++) sref = fmaxf(sref, hsb[k]);
            const float isref = sref > 0.0f ? __frcp_rn(sref) : 0.0f;
#pragma unroll 1
            for (int k = 0; k < 9; k++, h++) {
                const int st = h % C::S, bs = h % C::NBS;
                const uint32_t ratio = half2_bits(hsb[k] * isref);
                mbar_wait(&bempty[bs], ((h / C::NBS) & 1) ^ 1);
                mbar_wait(&lfull[st], (h / C::S) & 1);
                if (live) {
                    const unsigned char *lraw = ring + st * C::STAGE + C::BLK + (size_t)i * C::KCH * 16;
                    uint32_t w[C::N];
#pragma unroll
                    for (int c = 0; c < C::KCH; c++) *reinterpret_cast<uint4 *>(&w[4 * c]) = lds128(lraw + c * 16);
                    mbar_arrive(&lempty[st]);   // this thread is done with the stage's link record
#pragma unroll
                    for (int j = 0; j < C::N; j++) {
                        const uint32_t flip = (dagger && j >= NV) ? 0x80008000u : 0u;   // tau3 on the input
                        const uint32_t v = hmul2_u32(w[j] ^ flip, ratio);                // (re, im) * ratio
                        w[j] = part ? __byte_perm(v, 0, 0x1032) : (v ^ 0x80000000u);     // (im, re) | (re, -im)
                    }
                    const uint32_t a0 = tmem + lrow + C::ACOL + bs * C::ACOLS;
#pragma unroll
                    for (int u = 0; u < C::ACOLS / 16; u++) tmem_st16(a0 + 16 * u, w + 16 * u);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                } else {
                    mbar_arrive(&lempty[st]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&bfull[bs]);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 6-9)
        const int et = tid - 192, q = warp & 3, m = 32 * q + lane;
        const bool live = 32 * q < 2 * C::N;
        const int i = m >> 1, part = m & 1;
        const uint64_t pol_o = l2_policy_evict_first();
        const uint32_t lrow = (uint32_t)(32 * q) << 16;
        unsigned char *srow = stg + (m >> 3) * C::PITCH + ((i & 3) << 2) + part * 16;
        uint32_t t = 0;
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x, t++) {
            int rb;
            const int site = item_site(it, nrb, rb, sites);
            int x[4];
            decode(g, site, x);
            if (et < 9) es[et] = hop_scale<NV>(links, in, g, hl, x, site, et, nrb, rb);
            const int acc = t & 1;
            mbar_wait(&accfull[acc], (t >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            bar_named(2, 128);                              // es[] visible
            float sref = 0.0f;
#pragma unroll
            for (int k = 0; k < 9; k++) sref = fmaxf(sref, es[k]);
            const float sg = (dagger && i >= NV) ? -sref : sref;
            const uint32_t base = tmem + lrow + C::DCOL + acc * C::MR;
            // pass 1: the block's max |y| (D read twice: tensor memory is cheap to re-read)
            float mx = 0.0f;
            if (live) {
#pragma unroll
                for (int cb = 0; cb < C::MR / 32; cb++) {
                    uint32_t raw[32];
                    tmem_ld16_nowait(base + 32 * cb, raw);
                    tmem_ld16_nowait(base + 32 * cb + 16, raw + 16);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    reg_fence16(raw);
                    reg_fence16(raw + 16);
#pragma unroll
                    for (int j = 0; j < 32; j++) mx = fmaxf(mx, fabsf(__uint_as_float(raw[j]) * sg));
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) red[q] = mx;
            // the previous item's bulk stores must have read the staging tile
            if (et == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bar_named(2, 128);
            const float mb = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
            const float im = mb > 0.0f ? __frcp_rn(mb) : 0.0f;
            if (live) {
#pragma unroll
                for (int cb = 0; cb < C::MR / 32; cb++) {
                    uint32_t raw[32];
                    tmem_ld16_nowait(base + 32 * cb, raw);
                    tmem_ld16_nowait(base + 32 * cb + 16, raw + 16);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    reg_fence16(raw);
                    reg_fence16(raw + 16);
#pragma unroll
                    for (int p = 0; p < 16; p++) {
                        // lane pair (re, im) of output row i: the even lane stores column 2p, the odd
                        // lane column 2p + 1, each as one (re, im) half2 word
                        const float a = __uint_as_float(raw[2 * p]) * sg * im;
                        const float b = __uint_as_float(raw[2 * p + 1]) * sg * im;
                        const float o = __shfl_xor_sync(0xffffffffu, part ? a : b, 1);
                        __half2 hv = part ? __floats2half2_rn(o, b) : __floats2half2_rn(a, o);
                        *reinterpret_cast<uint32_t *>(srow + (32 * cb + 2 * p) * 16) =
                            *reinterpret_cast<uint32_t *>(&hv);
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[acc]);   // the MMA may reuse this accumulator
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_named(2, 128);
            if (et == 0) {
                unsigned char *blk = out + ((size_t)site * nrb + rb) * C::BLK;
#pragma unroll 1
                for (int c = 0; c < C::KCH; c++) bulk_s2g_hint(blk + c * C::LBO, stg + c * C::PITCH, C::LBO, pol_o);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                *reinterpret_cast<float4 *>(blk + C::A_BYTES) = make_float4(mb, 0.f, 0.f, 0.f);
            }
        }
        if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int NV>
static cudaError_t launch_mrhs_ts_t(const void *links, const void *in, void *out, const KGeom &g, int nrhs, int dagger,
                                    cudaStream_t s, int num_sms, const int *sites, int nsites, const MrhsHalo *halo)
{
    using C = MrhsTsCfg<NV>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(dslash_mrhs_ts<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int nrb = nrhs / C::MR;
    const int64_t items = (int64_t)(sites ? nsites : g.V) * nrb;
    if (items == 0) return cudaSuccess;
    MrhsHalo hl{};
    if (halo) hl = *halo;
    count_launch();
    const char *pfe = getenv("CD_MRHS_PF");
    const int pf = pfe ? atoi(pfe) : (NV == 32);
    dslash_mrhs_ts<NV><<<(unsigned)(items < num_sms ? items : num_sms), C::THREADS, C::SMEM, s>>>(
        static_cast<const unsigned char *>(links), static_cast<const unsigned char *>(in),
        static_cast<unsigned char *>(out), g, nrb, dagger, sites, nsites, hl, pf);
    return cudaGetLastError();
}

cudaError_t launch_mrhs(int nvec, const void *links, const void *in, void *out, const KGeom &g, int nrhs, int dagger,
                        cudaStream_t s, int num_sms, const int *sites, int nsites, const MrhsHalo *halo)
{
    if (nrhs % 128) return cudaErrorInvalidValue;
    // A/B switch: CD_MRHS_TS=1 = links as the A operand in tensor memory (dslash_mrhs_ts).  Parity-green
    // but 3-15 % slower than links as the shared-memory B operand (profiles/r02/mrhs_ts_ab.txt), so off.
    const char *tse = getenv("CD_MRHS_TS");
    if (tse && atoi(tse) == 1)
        return nvec == 24 ? launch_mrhs_ts_t<24>(links, in, out, g, nrhs, dagger, s, num_sms, sites, nsites, halo)
                          : launch_mrhs_ts_t<32>(links, in, out, g, nrhs, dagger, s, num_sms, sites, nsites, halo);
    // Nvec 24: two CTAs per SM, each a full pipeline (2 stages, 2 B slots, 79 registers): the kernel is
    // bound by the per-hop hand-offs of its single-thread roles, so two independent pipelines per SM
    // beat one deeper one -- 8^4 x 128 161.6 -> 152.1 us, 8^3x16 x 128 312 -> 300 us, 4^4 x 1024 (L2
    // resident) 86.3 -> 71.8 us (profiles/r02/mrhs_2cta_ab.txt).  CD_MRHS_2CTA=0: one CTA per SM.
    // Nvec 32 stays at one CTA (a 32 KB B slot leaves no room for two stages in half the SM).
    const char *c2 = getenv("CD_MRHS_2CTA");
    if (nvec == 24 && !(c2 && atoi(c2) == 0))
        return launch_mrhs_t<24, 2, 2>(links, in, out, g, nrhs, dagger, s, num_sms, sites, nsites, halo);
    // B slots: 3 for Nvec 24 (2 and 4 measured 1-3 % slower), 2 for Nvec 32 (shared memory)
    return nvec == 24 ? launch_mrhs_t<24, 3>(links, in, out, g, nrhs, dagger, s, num_sms, sites, nsites, halo)
                      : launch_mrhs_t<32, 2>(links, in, out, g, nrhs, dagger, s, num_sms, sites, nsites, halo);
}

// face blocks of every split dim -> send buffer (one CTA row per (mu, A/B), records [f][rb])
template <int BLK>
__global__ void mrhs_pack_kernel(const unsigned char *field, unsigned char *send, KGeom g, int4 pairs, int nrb,
                                 MrhsHalo offs)
{
    const int pi = blockIdx.y >> 1, blk = blockIdx.y & 1;
    const int mu = pi == 0 ? pairs.x : (pi == 1 ? pairs.y : (pi == 2 ? pairs.z : pairs.w));
    const int F = g.V / sel4(g.L, mu);
    int o3[3], n = 0;
    for (int nu = 0; nu < 4; nu++)
        if (nu != mu) o3[n++] = nu;
    for (int rec = blockIdx.x; rec < F * nrb; rec += gridDim.x) {
        const int f = rec / nrb, rb = rec - f * nrb;
        int x[4];
        int t = f;
        x[o3[0]] = t % g.L[o3[0]];
        t /= g.L[o3[0]];
        x[o3[1]] = t % g.L[o3[1]];
        x[o3[2]] = t / g.L[o3[1]];
        x[mu] = blk == 0 ? g.L[mu] - 1 : 0;
        const uint4 *src = reinterpret_cast<const uint4 *>(field + ((size_t)encode(g, x) * nrb + rb) * BLK);
        uint4 *dst = reinterpret_cast<uint4 *>(send + halo_off(offs, mu, blk) + (size_t)rec * BLK);
        for (int e = threadIdx.x; e < BLK / 16; e += blockDim.x) dst[e] = src[e];
    }
}

cudaError_t launch_mrhs_pack(int nvec, const void *field, void *send, const KGeom &g, int nrhs, const MrhsHalo &offs,
                             cudaStream_t s)
{
    int4 pairs = make_int4(0, 0, 0, 0);
    int np = 0;
    for (int mu = 0; mu < 4; mu++)
        if ((g.split >> mu) & 1) (&pairs.x)[np++] = mu;
    if (np == 0) return cudaSuccess;
    const dim3 grid(296, 2 * np);
    const unsigned char *f = static_cast<const unsigned char *>(field);
    unsigned char *d = static_cast<unsigned char *>(send);
    count_launch();
    if (nvec == 24) mrhs_pack_kernel<MrhsCfg<24>::BLK><<<grid, 256, 0, s>>>(f, d, g, pairs, nrhs / 128, offs);
    else mrhs_pack_kernel<MrhsCfg<32>::BLK><<<grid, 256, 0, s>>>(f, d, g, pairs, nrhs / 128, offs);
    return cudaGetLastError();
}

}  // namespace cd
