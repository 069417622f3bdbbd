// fields.cu -- data-movement kernels of the coarse-Dslash library (sm_100a):
// canonical <-> stored conversion of vectors and links (fp32 or binary16 + scale, DESIGN.md
// R12), the device synthetic-input generator (independent implementation of the
// counter-based splitmix64 recipe), and the bench L2-flush kernel.
#include <cuda_fp16.h>
#include <cstdint>

#include "cd_internal.h"
#include "device_common.cuh"

namespace cd {

// ------------------------------------------------------------------ quantisation (R12)
// s = max |x| over the record (fp32, exact); q = fp16_rn(fp32 x / s) with IEEE division;
// s == 0 -> q = +0.  Both roundings are round-to-nearest-even.
__device__ __forceinline__ __half2 quant2(float re, float im, float s)
{
    if (s > 0.0f) return __halves2half2(__float2half_rn(__fdiv_rn(re, s)), __float2half_rn(__fdiv_rn(im, s)));
    return __halves2half2(__float2half_rn(0.0f), __float2half_rn(0.0f));
}

template <int BS>
__device__ __forceinline__ float block_max(float m, float *red)
{
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, shfl_xor(m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < BS / 32; w++) s = fmaxf(s, red[w]);
    __syncthreads();
    return s;
}

__device__ __forceinline__ float2 load_canon(const void *src, int c128, size_t e)
{
    if (c128) {
        const double2 v = static_cast<const double2 *>(src)[e];
        return make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    return static_cast<const float2 *>(src)[e];
}

// canonical vector(s) [rhs][V][N] -> stored records [site][rhs]; one warp per record
__global__ void import_kernel(int fp16, int N, int64_t nsites, const void *src, int c128, unsigned char *dst, int nrhs)
{
    const int lane = threadIdx.x & 31;
    const int64_t site = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // record index
    if (site >= nsites * nrhs) return;
    const size_t base = ((size_t)(site % nrhs) * nsites + (size_t)(site / nrhs)) * N;
    if (!fp16) {
        float2 *o = reinterpret_cast<float2 *>(dst + (size_t)site * 8 * N);
        for (int i = lane; i < N; i += 32) o[i] = load_canon(src, c128, base + i);
        return;
    }
    float2 v[2];
    float m = 0.0f;
#pragma unroll
    for (int t = 0; t < 2; t++) {
        const int i = lane + 32 * t;
        v[t] = i < N ? load_canon(src, c128, base + i) : make_float2(0.f, 0.f);
        m = fmaxf(m, fmaxf(fabsf(v[t].x), fabsf(v[t].y)));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, shfl_xor(m, o));
    unsigned char *rec = dst + (size_t)site * (4 * N + 16);
#pragma unroll
    for (int t = 0; t < 2; t++) {
        const int i = lane + 32 * t;
        if (i < N) reinterpret_cast<__half2 *>(rec)[i] = quant2(v[t].x, v[t].y, m);
    }
    if (lane == 0) *reinterpret_cast<float *>(rec + 4 * N) = m;
}

// stored records [site][rhs] -> canonical vector(s) [rhs][V][N] (fp16: x = float(q) * s in fp32)
__global__ void export_kernel(int fp16, int N, int64_t nsites, const unsigned char *src, void *dst, int c128, int nrhs)
{
    const int lane = threadIdx.x & 31;
    const int64_t site = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // record index
    if (site >= nsites * nrhs) return;
    const size_t base = ((size_t)(site % nrhs) * nsites + (size_t)(site / nrhs)) * N;
    for (int i = lane; i < N; i += 32) {
        float2 v;
        if (!fp16) {
            v = reinterpret_cast<const float2 *>(src + (size_t)site * 8 * N)[i];
        } else {
            const unsigned char *rec = src + (size_t)site * (4 * N + 16);
            const float s = *reinterpret_cast<const float *>(rec + 4 * N);
            const __half2 q = reinterpret_cast<const __half2 *>(rec)[i];
            v = make_float2(__half2float(__low2half(q)) * s, __half2float(__high2half(q)) * s);
        }
        if (c128) static_cast<double2 *>(dst)[base + i] = make_double2(v.x, v.y);
        else static_cast<float2 *>(dst)[base + i] = v;
    }
}

// canonical matrices [nmats][N][N] -> stored matrix records; one CTA per matrix
template <int BS>
__global__ void __launch_bounds__(BS) links_convert_kernel(int fp16, int N, const void *src, int c128,
                                                           unsigned char *dst, int64_t mat0)
{
    __shared__ float red[BS / 32];
    const int64_t mat = mat0 + blockIdx.x;
    const int NN = N * N;
    const size_t base = (size_t)blockIdx.x * NN;   // src is the chunk starting at mat0
    if (!fp16) {
        float2 *o = reinterpret_cast<float2 *>(dst + (size_t)mat * 8 * NN);
        for (int e = threadIdx.x; e < NN; e += BS) o[e] = load_canon(src, c128, base + e);
        return;
    }
    float m = 0.0f;
    for (int e = threadIdx.x; e < NN; e += BS) {
        const float2 v = load_canon(src, c128, base + e);
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    const float s = block_max<BS>(m, red);
    unsigned char *rec = dst + (size_t)mat * (4 * NN + 16);
    for (int e = threadIdx.x; e < NN; e += BS) {
        const float2 v = load_canon(src, c128, base + e);
        reinterpret_cast<__half2 *>(rec)[e] = quant2(v.x, v.y, s);
    }
    if (threadIdx.x == 0) {
        float4 pad = make_float4(s, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4 *>(rec + 4 * NN) = pad;
    }
}

// ------------------------------------------------------------------ synthetic inputs
// splitmix64 over GLOBAL indices; u = ((h >> 42) - 2^21) * 2^-21, exact in fp32.
__device__ __forceinline__ uint64_t splitmix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float hash_u(uint64_t base, uint64_t ctr)
{
    const uint64_t h = splitmix(base + ctr);
    const int q = (int)(h >> 42) - (1 << 21);
    return (float)q * 0x1p-21f;
}

struct GenGeom {
    int Lloc[4], Lg[4], origin[4];
};

__device__ __forceinline__ void local_to_global(const GenGeom &g, int64_t s, int xg[4])
{
    int64_t t = s;
    for (int mu = 0; mu < 4; mu++) {
        xg[mu] = (int)(t % g.Lloc[mu]) + g.origin[mu];
        t /= g.Lloc[mu];
    }
}
__device__ __forceinline__ int64_t gindex(const GenGeom &g, const int xg[4])
{
    return (((int64_t)xg[3] * g.Lg[2] + xg[2]) * g.Lg[1] + xg[1]) * g.Lg[0] + xg[0];
}

// G(gsite, k)[i][j] (re, im)
__device__ __forceinline__ float2 rawG(uint64_t base, int64_t gsite, int k, int i, int j, int N)
{
    const uint64_t c = ((((uint64_t)gsite * 9 + k) * N + i) * N + j) * 2;
    return make_float2(hash_u(base, c), hash_u(base, c + 1));
}

// Link value of recipe `kind` (see cd_links_kind) at local site s, hop k, entry (i, j).
__device__ __forceinline__ float2 link_value(const GenGeom &g, uint64_t base, int kind, int64_t s, int k, int i, int j,
                                             int N, float scale)
{
    const bool ti = kind >= 2, herm = (kind & 1);
    int xg[4];
    local_to_global(g, s, xg);
    const int64_t gs = ti ? 0 : gindex(g, xg);
    float2 v;
    if (!herm || (k != 8 && (k & 1) == 0)) {
        v = rawG(base, gs, k, i, j, N);
    } else {
        const int nv = N / 2;
        const float ss = ((i < nv) == (j < nv)) ? 1.0f : -1.0f;
        if (k == 8) {
            const float2 a = rawG(base, gs, 8, i, j, N), b = rawG(base, gs, 8, j, i, N);
            v = make_float2(0.5f * (a.x + ss * b.x), 0.5f * (a.y + ss * (-b.y)));
        } else {
            const int mu = k >> 1;
            int xb[4] = {xg[0], xg[1], xg[2], xg[3]};
            xb[mu] = (xb[mu] - 1 + g.Lg[mu]) % g.Lg[mu];
            const int64_t gb = ti ? 0 : gindex(g, xb);
            const float2 b = rawG(base, gb, 2 * mu, j, i, N);
            v = make_float2(ss * b.x, ss * (-b.y));
        }
    }
    return make_float2(v.x * scale, v.y * scale);
}

template <int BS>
__global__ void __launch_bounds__(BS) links_generate_kernel(int fp16, int N, GenGeom g, uint64_t base, int kind,
                                                            float scale, unsigned char *dst)
{
    __shared__ float red[BS / 32];
    const int64_t mat = blockIdx.x;
    const int64_t s = mat / 9;
    const int k = (int)(mat - s * 9);
    const int NN = N * N;
    if (!fp16) {
        float2 *o = reinterpret_cast<float2 *>(dst + (size_t)mat * 8 * NN);
        for (int e = threadIdx.x; e < NN; e += BS) o[e] = link_value(g, base, kind, s, k, e / N, e % N, N, scale);
        return;
    }
    float m = 0.0f;
    for (int e = threadIdx.x; e < NN; e += BS) {
        const float2 v = link_value(g, base, kind, s, k, e / N, e % N, N, scale);
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    const float sc = block_max<BS>(m, red);
    unsigned char *rec = dst + (size_t)mat * (4 * NN + 16);
    for (int e = threadIdx.x; e < NN; e += BS) {
        const float2 v = link_value(g, base, kind, s, k, e / N, e % N, N, scale);
        reinterpret_cast<__half2 *>(rec)[e] = quant2(v.x, v.y, sc);
    }
    if (threadIdx.x == 0) *reinterpret_cast<float4 *>(rec + 4 * NN) = make_float4(sc, 0.f, 0.f, 0.f);
}

// one warp per record [site][rhs]; right-hand side r uses tag + r
__global__ void field_generate_kernel(int fp16, int N, int64_t nsites, GenGeom g, uint64_t seed, uint32_t tag,
                                      float scale, unsigned char *dst, int nrhs)
{
    const int lane = threadIdx.x & 31;
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (e >= nsites * nrhs) return;
    const int64_t s = e / nrhs;
    const uint64_t base = splitmix(seed ^ ((uint64_t)(tag + (uint32_t)(e % nrhs)) << 56));
    int xg[4];
    local_to_global(g, s, xg);
    const int64_t gs = gindex(g, xg);
    float2 v[2];
    float m = 0.0f;
#pragma unroll
    for (int t = 0; t < 2; t++) {
        const int i = lane + 32 * t;
        if (i < N) {
            const uint64_t c = ((uint64_t)gs * N + i) * 2;
            v[t] = make_float2(hash_u(base, c) * scale, hash_u(base, c + 1) * scale);
        } else {
            v[t] = make_float2(0.f, 0.f);
        }
        m = fmaxf(m, fmaxf(fabsf(v[t].x), fabsf(v[t].y)));
    }
    if (!fp16) {
        float2 *o = reinterpret_cast<float2 *>(dst + (size_t)e * 8 * N);
#pragma unroll
        for (int t = 0; t < 2; t++)
            if (lane + 32 * t < N) o[lane + 32 * t] = v[t];
        return;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, shfl_xor(m, o));
    unsigned char *rec = dst + (size_t)e * (4 * N + 16);
#pragma unroll
    for (int t = 0; t < 2; t++)
        if (lane + 32 * t < N) reinterpret_cast<__half2 *>(rec)[lane + 32 * t] = quant2(v[t].x, v[t].y, m);
    if (lane == 0) *reinterpret_cast<float4 *>(rec + 4 * N) = make_float4(m, 0.f, 0.f, 0.f);
}

// ------------------------------------------------------------------ tensor-core multi-RHS fp16 layout (R22)
// block (site, rb) = 128 right-hand sides: [K chunk c][rhs r][4 half2] + fp32 scale (16 B);
// one scale per block: s = max |x| over its 128 x N complex values, q = fp16_rn(x / s).
__device__ __forceinline__ size_t tc_off(int N, int r, int i)   // byte offset of complex i of rhs r
{
    return (size_t)(i >> 2) * 2048 + (size_t)r * 16 + (size_t)(i & 3) * 4;
}

// canonical [rhs][V][N] -> blocks; one CTA per (site, block)
__global__ void __launch_bounds__(256) tc_import_kernel(int N, int64_t nsites, int nrb, const void *src, int c128,
                                                        unsigned char *dst)
{
    __shared__ float red[8];
    const int64_t site = blockIdx.x / nrb;
    const int rb = (int)(blockIdx.x - site * nrb);
    const int n = 128 * N;
    auto idx = [&](int e) { return ((size_t)(rb * 128 + e / N) * nsites + site) * N + (e % N); };
    float m = 0.0f;
    for (int e = threadIdx.x; e < n; e += 256) {
        const float2 v = load_canon(src, c128, idx(e));
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    const float sc = block_max<256>(m, red);
    unsigned char *blk = dst + (size_t)blockIdx.x * (128 * 4 * N + 16);
    for (int e = threadIdx.x; e < n; e += 256) {
        const float2 v = load_canon(src, c128, idx(e));
        *reinterpret_cast<__half2 *>(blk + tc_off(N, e / N, e % N)) = quant2(v.x, v.y, sc);
    }
    if (threadIdx.x == 0) *reinterpret_cast<float4 *>(blk + 128 * 4 * N) = make_float4(sc, 0.f, 0.f, 0.f);
}

__global__ void __launch_bounds__(256) tc_export_kernel(int N, int64_t nsites, int nrb, const unsigned char *src,
                                                        void *dst, int c128)
{
    const int64_t site = blockIdx.x / nrb;
    const int rb = (int)(blockIdx.x - site * nrb);
    const unsigned char *blk = src + (size_t)blockIdx.x * (128 * 4 * N + 16);
    const float sc = *reinterpret_cast<const float *>(blk + 128 * 4 * N);
    for (int e = threadIdx.x; e < 128 * N; e += 256) {
        const int r = e / N, i = e % N;
        const __half2 q = *reinterpret_cast<const __half2 *>(blk + tc_off(N, r, i));
        const float2 v = make_float2(__half2float(__low2half(q)) * sc, __half2float(__high2half(q)) * sc);
        const size_t o = ((size_t)(rb * 128 + r) * nsites + site) * N + i;
        if (c128) static_cast<double2 *>(dst)[o] = make_double2(v.x, v.y);
        else static_cast<float2 *>(dst)[o] = v;
    }
}

// generator values of right-hand side (tag + r) quantised per block
__global__ void __launch_bounds__(256) tc_generate_kernel(int N, int nrb, GenGeom g, uint64_t seed, uint32_t tag,
                                                          float scale, unsigned char *dst)
{
    __shared__ float red[8];
    const int64_t site = blockIdx.x / nrb;
    const int rb = (int)(blockIdx.x - site * nrb);
    int xg[4];
    local_to_global(g, site, xg);
    const int64_t gs = gindex(g, xg);
    auto val = [&](int e) {
        const int r = rb * 128 + e / N, i = e % N;
        const uint64_t base = splitmix(seed ^ ((uint64_t)(tag + (uint32_t)r) << 56));
        const uint64_t c = ((uint64_t)gs * N + i) * 2;
        return make_float2(hash_u(base, c) * scale, hash_u(base, c + 1) * scale);
    };
    float m = 0.0f;
    for (int e = threadIdx.x; e < 128 * N; e += 256) {
        const float2 v = val(e);
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    const float sc = block_max<256>(m, red);
    unsigned char *blk = dst + (size_t)blockIdx.x * (128 * 4 * N + 16);
    for (int e = threadIdx.x; e < 128 * N; e += 256) {
        const float2 v = val(e);
        *reinterpret_cast<__half2 *>(blk + tc_off(N, e / N, e % N)) = quant2(v.x, v.y, sc);
    }
    if (threadIdx.x == 0) *reinterpret_cast<float4 *>(blk + 128 * 4 * N) = make_float4(sc, 0.f, 0.f, 0.f);
}

__global__ void flush_kernel(uint4 *buf, size_t n)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

// ------------------------------------------------------------------ host launchers
static uint64_t host_splitmix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static GenGeom gen_geom(const cd_context *ctx)
{
    GenGeom g;
    for (int mu = 0; mu < 4; mu++) {
        g.Lloc[mu] = ctx->local[mu];
        g.Lg[mu] = ctx->geom.global_dims[mu];
        g.origin[mu] = ctx->coords[mu] * ctx->local[mu];
    }
    return g;
}

cudaError_t launch_import(cd_precision p, int nvec, int64_t nsites, const void *src, int src_c128, void *dst,
                          cudaStream_t s, int nrhs)
{
    if (nsites == 0) return cudaSuccess;
    count_launch();
    if (p == CD_FP16 && nrhs > 1) {
        tc_import_kernel<<<(unsigned)(nsites * (nrhs / 128)), 256, 0, s>>>(2 * nvec, nsites, nrhs / 128, src, src_c128,
                                                                           static_cast<unsigned char *>(dst));
        return cudaGetLastError();
    }
    import_kernel<<<(unsigned)((nsites * nrhs + 7) / 8), 256, 0, s>>>(p == CD_FP16, 2 * nvec, nsites, src, src_c128,
                                                                         static_cast<unsigned char *>(dst), nrhs);
    return cudaGetLastError();
}

cudaError_t launch_export(cd_precision p, int nvec, int64_t nsites, const void *src, void *dst, int dst_c128,
                          cudaStream_t s, int nrhs)
{
    if (nsites == 0) return cudaSuccess;
    count_launch();
    if (p == CD_FP16 && nrhs > 1) {
        tc_export_kernel<<<(unsigned)(nsites * (nrhs / 128)), 256, 0, s>>>(
            2 * nvec, nsites, nrhs / 128, static_cast<const unsigned char *>(src), dst, dst_c128);
        return cudaGetLastError();
    }
    export_kernel<<<(unsigned)((nsites * nrhs + 7) / 8), 256, 0, s>>>(
        p == CD_FP16, 2 * nvec, nsites, static_cast<const unsigned char *>(src), dst, dst_c128, nrhs);
    return cudaGetLastError();
}

cudaError_t launch_links_convert(cd_precision p, int nvec, int64_t nmats, const void *src, int src_c128, void *dst,
                                 cudaStream_t s, int64_t mat0)
{
    if (nmats == 0) return cudaSuccess;
    count_launch();
    links_convert_kernel<256><<<(unsigned)nmats, 256, 0, s>>>(p == CD_FP16, 2 * nvec, src, src_c128,
                                                               static_cast<unsigned char *>(dst), mat0);
    return cudaGetLastError();
}

cudaError_t launch_links_generate(cd_precision p, int nvec, const cd_context *ctx, int kind, uint64_t seed,
                                  int scale_log2, void *dst, cudaStream_t s)
{
    const uint64_t tag = (kind >= 2) ? 4 : 1;
    const uint64_t base = host_splitmix(seed ^ (tag << 56));
    count_launch();
    links_generate_kernel<256><<<(unsigned)(ctx->V * 9), 256, 0, s>>>(p == CD_FP16, 2 * nvec, gen_geom(ctx), base,
                                                                      kind, ldexpf(1.0f, scale_log2),
                                                                      static_cast<unsigned char *>(dst));
    return cudaGetLastError();
}

cudaError_t launch_field_generate(cd_precision p, int nvec, const cd_context *ctx, uint64_t seed, uint32_t tag,
                                  int scale_log2, void *dst, cudaStream_t s, int nrhs)
{
    count_launch();
    if (p == CD_FP16 && nrhs > 1) {
        tc_generate_kernel<<<(unsigned)(ctx->V * (nrhs / 128)), 256, 0, s>>>(
            2 * nvec, nrhs / 128, gen_geom(ctx), seed, tag, ldexpf(1.0f, scale_log2), static_cast<unsigned char *>(dst));
        return cudaGetLastError();
    }
    field_generate_kernel<<<(unsigned)((ctx->V * nrhs + 7) / 8), 256, 0, s>>>(
        p == CD_FP16, 2 * nvec, ctx->V, gen_geom(ctx), seed, tag, ldexpf(1.0f, scale_log2),
        static_cast<unsigned char *>(dst), nrhs);
    return cudaGetLastError();
}

cudaError_t launch_flush(void *buf, size_t bytes, cudaStream_t s)
{
    count_launch();
    flush_kernel<<<148 * 8, 256, 0, s>>>(static_cast<uint4 *>(buf), bytes / 16);
    return cudaGetLastError();
}

}  // namespace cd
