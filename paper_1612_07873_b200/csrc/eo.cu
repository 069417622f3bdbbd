// eo.cu -- even-odd (red-black) preconditioned coarse operator (§3.3,
// used "on all levels"):
//
//     M_ee v_e = X_e v_e - D_eo X_o^{-1} D_oe v_e           (Schur complement on even sites)
//
// Setup (coarse_links_prepare_eo): for every odd site o, X_o^{-1} by Gauss-Jordan with partial
// pivoting in fp64 in shared memory, then L'_k(o) = X_o^{-1} L_k(o) for the 8 hops (fp64 products,
// stored fp32); even sites keep their 9 matrices.  Apply = two parity-restricted hop kernels:
//
//     A (odd sites):   t_o = sum_k L'_k(o) v_e(nbr_k(o))                 (8 matrices per site)
//     B (even sites):  y_e = X_e v_e - sum_k L_k(e) t_o(nbr_k(e))        (9 matrices per site)
//
// Half fields hold the V/2 sites of one parity in half-index order h = s >> 1 (every L_mu even,
// so consecutive x0 pairs hold one site of each parity).  fp32 storage.  The dagger of a
// tau3-hermitian operator is tau3 M_ee tau3 (tests/test_oracle_eo.py): input sign flips in A and in
// the X term of B, output flips in B.
#include <cuda_fp16.h>
#include <cstdint>

#include "cd_internal.h"
#include "device_common.cuh"

namespace cd {

// site of parity p with half index h
__device__ __forceinline__ int parity_site(const KGeom &g, int h, int p)
{
    int x[4];
    decode(g, 2 * h, x);
    return 2 * h + (((x[1] + x[2] + x[3]) & 1) != p ? 1 : 0);
}

__device__ __forceinline__ bool eo_is_face(const KGeom &g, const int x[4])
{
#pragma unroll
    for (int mu = 0; mu < 4; mu++)
        if (((g.split >> mu) & 1) && (x[mu] == 0 || x[mu] == g.L[mu] - 1)) return true;
    return false;
}

// ------------------------------------------------------------------ setup: X_o^{-1} L_k(o)
template <int NV>
__global__ void __launch_bounds__(256) eo_prepare_odd(const unsigned char *full, unsigned char *odd_out, KGeom g,
                                                      int *singular)
{
    constexpr int N = 2 * NV;
    constexpr int W = 2 * N;                        // augmented width
    extern __shared__ __align__(16) double2 sm[];  // [N][2N] augmented, then [N] column copy
    double2 *M = sm;
    double2 *col = sm + N * W;
    __shared__ int piv;
    const int h = blockIdx.x;
    const int s = parity_site(g, h, 1);
    const float2 *X = reinterpret_cast<const float2 *>(full + ((size_t)s * 9 + 8) * (8 * N * N));
    for (int e = threadIdx.x; e < N * W; e += blockDim.x) {
        const int i = e / W, j = e - i * W;
        M[e] = j < N ? make_double2(X[i * N + j].x, X[i * N + j].y) : make_double2(j - N == i ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    for (int c = 0; c < N; c++) {
        if (threadIdx.x < 32) {   // pivot: largest |M[i][c]|, i >= c
            double best = -1.0;
            int bi = c;
            for (int i = c + threadIdx.x; i < N; i += 32) {
                const double2 v = M[i * W + c];
                const double a = v.x * v.x + v.y * v.y;
                if (a > best) best = a, bi = i;
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) best = ob, bi = oi;
            }
            if (threadIdx.x == 0) {
                piv = bi;
                if (best == 0.0) atomicExch(singular, 1);
            }
        }
        __syncthreads();
        const int p = piv;
        if (p != c)
            for (int j = threadIdx.x; j < W; j += blockDim.x) {
                const double2 t = M[c * W + j];
                M[c * W + j] = M[p * W + j];
                M[p * W + j] = t;
            }
        __syncthreads();
        const double2 pv = M[c * W + c];
        const double den = pv.x * pv.x + pv.y * pv.y;
        const double2 inv = den > 0.0 ? make_double2(pv.x / den, -pv.y / den) : make_double2(0.0, 0.0);
        __syncthreads();
        for (int j = threadIdx.x; j < W; j += blockDim.x) {   // normalise the pivot row
            const double2 a = M[c * W + j];
            M[c * W + j] = make_double2(a.x * inv.x - a.y * inv.y, a.x * inv.y + a.y * inv.x);
        }
        for (int i = threadIdx.x; i < N; i += blockDim.x) col[i] = M[i * W + c];
        __syncthreads();
        for (int e = threadIdx.x; e < N * W; e += blockDim.x) {   // eliminate column c elsewhere
            const int i = e / W, j = e - i * W;
            if (i == c) continue;
            const double2 f = col[i], b = M[c * W + j];
            M[e] = make_double2(M[e].x - (f.x * b.x - f.y * b.y), M[e].y - (f.x * b.y + f.y * b.x));
        }
        __syncthreads();
    }
    // L'_k = X^{-1} L_k for k = 0..7 (fp64 accumulation), stored fp32
    for (int k = 0; k < 8; k++) {
        const float2 *Lk = reinterpret_cast<const float2 *>(full + ((size_t)s * 9 + k) * (8 * N * N));
        float2 *out = reinterpret_cast<float2 *>(odd_out + ((size_t)h * 8 + k) * (8 * N * N));
        for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
            const int i = e / N, j = e - i * N;
            double re = 0.0, im = 0.0;
            for (int m = 0; m < N; m++) {
                const double2 a = M[i * W + N + m];
                const float2 b = Lk[m * N + j];
                re += a.x * b.x - a.y * b.y;
                im += a.x * b.y + a.y * b.x;
            }
            out[e] = make_float2((float)re, (float)im);
        }
    }
}

// even sites: their 9 matrices in half order
template <int NV>
__global__ void eo_copy_even(const unsigned char *full, unsigned char *even_out, KGeom g)
{
    constexpr int MREC = 8 * (2 * NV) * (2 * NV);
    const int h = blockIdx.x / 9, k = blockIdx.x - (blockIdx.x / 9) * 9;
    const int s = parity_site(g, h, 0);
    const uint4 *src = reinterpret_cast<const uint4 *>(full + ((size_t)s * 9 + k) * MREC);
    uint4 *dst = reinterpret_cast<uint4 *>(even_out + ((size_t)h * 9 + k) * MREC);
    for (int e = threadIdx.x; e < MREC / 16; e += blockDim.x) dst[e] = src[e];
}

// ------------------------------------------------------------------ parity hop kernel
// MODE 0 (A, odd sites):  out = sum_{k<8} L'_k in_hop(nbr_k)          links: [h][8]
// MODE 1 (B, even sites): out = X in_self - sum_{k<8} L_k in_hop(nbr_k)  links: [h][9] (X = record 8)
// CTA = (half site, 16 rows); warp w = hop (9 warps; MODE 0 idles warp 8); lanes = (4 rows x 8 chunks),
// 4 row groups per warp.  fp32.
template <int NV, int MODE>
__global__ void __launch_bounds__(288) dslash_parity(const unsigned char *__restrict__ links, const unsigned char *in_self,
                                                     const unsigned char *in_hop, unsigned char *out, KGeom g, int dagger,
                                                     int halo, float2 *scratch)
{
    using Q = Cfg<CD_FP32, NV>;
    constexpr int ROWS = 16, NRB = Q::N / ROWS, RG = ROWS / Q::R;
    constexpr int NM = MODE == 0 ? 8 : 9;
    constexpr int P = MODE == 0 ? 1 : 0;   // parity of the output sites
    __shared__ __align__(16) unsigned char vs[9 * Q::VREC];
    __shared__ float2 part[9][ROWS];
    const int h = blockIdx.x / NRB, rb = blockIdx.x - (blockIdx.x / NRB) * NRB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = kseq(warp);   // 8 (X) first, then 0..7
    const int r = lane / Q::D, d = lane % Q::D;
    const int s = parity_site(g, h, P);
    int x[4];
    decode(g, s, x);
    // multi-rank: remote hops are added by eo_halo once the exchange has landed
    const bool active = ((MODE == 1) || (k != 8)) && !(halo && remote_hop(g, x, k));
    uint4 Lc[RG][Q::C];
    if (active) {
        const int rec = (k == 8) ? 8 : k;
        const unsigned char *m = links + ((size_t)h * NM + rec) * Q::MREC;
#pragma unroll
        for (int gg = 0; gg < RG; gg++)
#pragma unroll
            for (int c = 0; c < Q::C; c++)
                Lc[gg][c] = ld_stream(m + (rb * ROWS + gg * Q::R + r) * Q::ROWB + (d + Q::D * c) * 16);
    }
    pdl_trigger();
    pdl_wait();
    for (int t = threadIdx.x; t < 9 * Q::VCH; t += 288) {   // the 9 input records (half indices)
        const int kk = t / Q::VCH, e = t - kk * Q::VCH;
        if (kk == 8 && MODE == 0) continue;
        if (halo && remote_hop(g, x, kk)) continue;
        const unsigned char *src = kk == 8 ? in_self + (size_t)h * Q::VREC
                                           : in_hop + (size_t)(neighbour(g, x, s, kk) >> 1) * Q::VREC;
        *reinterpret_cast<uint4 *>(vs + kk * Q::VREC + e * 16) = ld_nc(src + e * 16);
    }
    __syncthreads();
    if (active) {
        // input tau3 (dagger): the v_e inputs -- all hops in A, the X term in B
        const bool flip_in = dagger && (MODE == 0 || k == 8);
        const float hs = (MODE == 1 && k != 8) ? -1.0f : 1.0f;
#pragma unroll
        for (int gg = 0; gg < RG; gg++) {
            float re = 0.0f, im = 0.0f;
#pragma unroll
            for (int c = 0; c < Q::C; c++) {
                const int q = d + Q::D * c;
                uint4 vq = lds128(vs + k * Q::VREC + q * 16);
                if (flip_in && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
                cmac2(Lc[gg][c], vq, re, im);
            }
#pragma unroll
            for (int o = Q::D / 2; o >= 1; o >>= 1) {
                re += shfl_xor(re, o);
                im += shfl_xor(im, o);
            }
            if (d == 0) part[warp][gg * Q::R + r] = make_float2(hs * re, hs * im);
        }
    } else if (d == 0) {
#pragma unroll
        for (int gg = 0; gg < RG; gg++) part[warp][gg * Q::R + r] = make_float2(0.0f, 0.0f);
    }
    __syncthreads();
    if (threadIdx.x < ROWS) {
        float yr = 0.0f, yi = 0.0f;
#pragma unroll
        for (int w = (MODE == 0 ? 1 : 0); w < 9; w++) {
            yr += part[w][threadIdx.x].x;
            yi += part[w][threadIdx.x].y;
        }
        const int row = rb * ROWS + threadIdx.x;
        if (halo && eo_is_face(g, x)) {   // partial (no output sign yet) for eo_halo
            scratch[(size_t)s * Q::N + row] = make_float2(yr, yi);
        } else {
            const float sg = (MODE == 1 && dagger && row >= NV) ? -1.0f : 1.0f;
            reinterpret_cast<float2 *>(out + (size_t)h * Q::VREC)[row] = make_float2(sg * yr, sg * yi);
        }
    }
}

// ------------------------------------------------------------------ multi-rank halo pieces
// The half fields travel in the full-field wire format (R13): face records of the
// other parity are simply not written (never read), so the plan, buffers and NCCL exchange of
// the full operator are reused unchanged.
template <int NV>
__global__ void eo_pack(const unsigned char *half, PackDst d, KGeom g, int4 pairs, int parity)
{
    using Q = Cfg<CD_FP32, NV>;
    constexpr int PREC = 8 * Q::N, CPR = PREC / 16;
    const int mu = (&pairs.x)[blockIdx.y >> 1], blk = blockIdx.y & 1;
    const int F = g.F[mu];
    int o3[3], n = 0;
    for (int nu = 0; nu < 4; nu++)
        if (nu != mu) o3[n++] = nu;
    unsigned char *dst = d.dst[mu][blk];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < F * CPR; e += gridDim.x * blockDim.x) {
        const int f = e / CPR, ch = e - f * CPR;
        int x[4];
        int t = f;
        x[o3[0]] = t % g.L[o3[0]];
        t /= g.L[o3[0]];
        x[o3[1]] = t % g.L[o3[1]];
        x[o3[2]] = t / g.L[o3[1]];
        x[mu] = blk == 0 ? g.L[mu] - 1 : 0;
        if (((x[0] + x[1] + x[2] + x[3]) & 1) != parity) continue;
        const unsigned char *rec = half + (size_t)(encode(g, x) >> 1) * Q::VREC;
        *reinterpret_cast<uint4 *>(dst + (size_t)f * PREC + ch * 16) = *reinterpret_cast<const uint4 *>(rec + ch * 16);
    }
    signal_block(d.flag[mu][blk]);
}

// one CTA per face site of the output parity: partial + the remote hops, then the final store
template <int NV, int MODE>
__global__ void __launch_bounds__(32 * (2 * NV / 4)) eo_halo(const unsigned char *__restrict__ links,
                                                              const unsigned char *__restrict__ recv,
                                                              const int *face_sites, const float2 *scratch,
                                                              unsigned char *out, KGeom g, int dagger)
{
    using Q = Cfg<CD_FP32, NV>;
    constexpr int NM = MODE == 0 ? 8 : 9;
    constexpr int P = MODE == 0 ? 1 : 0;
    constexpr int PREC = 8 * Q::N;
    const int s = face_sites[blockIdx.x];
    int x[4];
    decode(g, s, x);
    if (((x[0] + x[1] + x[2] + x[3]) & 1) != P) return;
    const int h = s >> 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = lane / Q::D, d = lane % Q::D;
    const int row = warp * Q::R + r;
    float re = 0.0f, im = 0.0f;
    for (int k = 0; k < 8; k++) {
        if (!remote_hop(g, x, k)) continue;
        const int mu = k >> 1;
        const int blk = (k & 1) ? 0 : 1;   // +mu hop: block B of the +mu neighbour; -mu hop: block A
        int o3[3], n = 0;
        for (int nu = 0; nu < 4; nu++)
            if (nu != mu) o3[n++] = nu;
        const int f = (x[o3[2]] * g.L[o3[1]] + x[o3[1]]) * g.L[o3[0]] + x[o3[0]];
        const unsigned char *vrec = recv + g.blk_off[mu][blk] + (size_t)f * PREC;
        const unsigned char *m = links + ((size_t)h * NM + k) * Q::MREC;
#pragma unroll
        for (int c = 0; c < Q::C; c++) {
            const int q = d + Q::D * c;
            uint4 vq = ld_nc(vrec + q * 16);
            if (MODE == 0 && dagger && q * Q::CPC >= NV) vq = neg_chunk<false>(vq);
            cmac2(ld_nc(m + row * Q::ROWB + q * 16), vq, re, im);
        }
    }
#pragma unroll
    for (int o = Q::D / 2; o >= 1; o >>= 1) {
        re += shfl_xor(re, o);
        im += shfl_xor(im, o);
    }
    if (d == 0) {
        const float2 p = scratch[(size_t)s * Q::N + row];
        const float hs = MODE == 1 ? -1.0f : 1.0f;
        const float sg = (MODE == 1 && dagger && row >= NV) ? -1.0f : 1.0f;
        reinterpret_cast<float2 *>(out + (size_t)h * Q::VREC)[row] =
            make_float2(sg * (p.x + hs * re), sg * (p.y + hs * im));
    }
}

// ------------------------------------------------------------------ launchers
template <int NV>
static cudaError_t eo_prepare_t(const void *full, void *even, void *odd, const KGeom &g, int *singular, cudaStream_t s)
{
    constexpr int N = 2 * NV;
    const size_t smem = sizeof(double2) * (size_t)(N * 2 * N + N);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(eo_prepare_odd<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    count_launch(2);
    eo_copy_even<NV><<<(unsigned)(g.V / 2 * 9), 256, 0, s>>>(static_cast<const unsigned char *>(full),
                                                             static_cast<unsigned char *>(even), g);
    eo_prepare_odd<NV><<<(unsigned)(g.V / 2), 256, smem, s>>>(static_cast<const unsigned char *>(full),
                                                              static_cast<unsigned char *>(odd), g, singular);
    return cudaGetLastError();
}

cudaError_t launch_eo_prepare(int nvec, const void *full, void *even, void *odd, const KGeom &g, int *singular,
                              cudaStream_t s)
{
    return nvec == 24 ? eo_prepare_t<24>(full, even, odd, g, singular, s) : eo_prepare_t<32>(full, even, odd, g, singular, s);
}

template <int NV>
static cudaError_t eo_mode_launch(int mode, const unsigned char *links, const unsigned char *self, const unsigned char *hop,
                                  unsigned char *out, const KGeom &g, int dagger, int halo, float2 *scratch,
                                  cudaStream_t s, bool pdl)
{
    constexpr int NRB = 2 * NV / 16;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(g.V / 2 * NRB));
    cfg.blockDim = dim3(288);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KGeom gg = g;
    int dg = dagger, hl = halo;
    void *args[] = {&links, &self, &hop, &out, &gg, &dg, &hl, &scratch};
    count_launch();
    return cudaLaunchKernelExC(&cfg, mode == 0 ? (const void *)dslash_parity<NV, 0> : (const void *)dslash_parity<NV, 1>,
                               args);
}

template <int NV>
static cudaError_t eo_apply_t(const EoApply &e)
{
    const unsigned char *ev = static_cast<const unsigned char *>(e.even), *od = static_cast<const unsigned char *>(e.odd);
    const unsigned char *vi = static_cast<const unsigned char *>(e.in_e);
    unsigned char *t = static_cast<unsigned char *>(e.t_o), *y = static_cast<unsigned char *>(e.out_e);
    if (!e.halo) {
        cudaError_t r = eo_mode_launch<NV>(0, od, nullptr, vi, t, e.g, e.dagger, 0, nullptr, e.s, e.pdl);
        if (r != cudaSuccess) return r;
        return eo_mode_launch<NV>(1, ev, vi, t, y, e.g, e.dagger, 0, nullptr, e.s, e.pdl);
    }
    // multi-rank: per mode, pack + exchange (comm stream) overlap the interior kernel; the halo
    // kernel adds the remote hops of the face sites once the exchange landed.
    int4 pairs = make_int4(0, 0, 0, 0);
    int np = 0;
    for (int mu = 0; mu < 4; mu++)
        if ((e.g.split >> mu) & 1) (&pairs.x)[np++] = mu;
    for (int mode = 0; mode < 2; mode++) {
        const unsigned char *src = mode == 0 ? vi : t;   // the half field the hops read
        PackDst pd;
        const void *recv = nullptr;
        cudaError_t r = e.begin(e.exchange_arg, &pd, &recv);
        if (r == cudaSuccess) r = cudaEventRecord(e.ev_in, e.s);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(e.comm_stream, e.ev_in, 0);
        if (r != cudaSuccess) return r;
        count_launch();
        eo_pack<NV><<<dim3(kPutCtas, 2 * np), 256, 0, e.comm_stream>>>(src, pd, e.g, pairs, mode == 0 ? 0 : 1);
        if ((r = cudaGetLastError()) != cudaSuccess) return r;
        if ((r = e.post(e.exchange_arg)) != cudaSuccess) return r;
        if ((r = cudaEventRecord(e.ev_halo, e.comm_stream)) != cudaSuccess) return r;
        r = mode == 0 ? eo_mode_launch<NV>(0, od, nullptr, vi, t, e.g, e.dagger, 1, e.scratch, e.s, false)
                      : eo_mode_launch<NV>(1, ev, vi, t, y, e.g, e.dagger, 1, e.scratch, e.s, false);
        if (r != cudaSuccess) return r;
        if ((r = cudaStreamWaitEvent(e.s, e.ev_halo, 0)) != cudaSuccess) return r;
        if ((r = e.finish(e.exchange_arg)) != cudaSuccess) return r;
        count_launch();
        const unsigned char *rv = static_cast<const unsigned char *>(recv);
        if (mode == 0)
            eo_halo<NV, 0><<<e.n_face, 32 * (2 * NV / 4), 0, e.s>>>(od, rv, e.face_sites, e.scratch, t, e.g, e.dagger);
        else
            eo_halo<NV, 1><<<e.n_face, 32 * (2 * NV / 4), 0, e.s>>>(ev, rv, e.face_sites, e.scratch, y, e.g, e.dagger);
        if ((r = cudaGetLastError()) != cudaSuccess) return r;
    }
    return cudaSuccess;
}

cudaError_t launch_eo_apply(int nvec, const EoApply &e)
{
    return nvec == 24 ? eo_apply_t<24>(e) : eo_apply_t<32>(e);
}

}  // namespace cd
