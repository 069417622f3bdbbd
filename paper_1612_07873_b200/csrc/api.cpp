// api.cpp -- C ABI of the coarse-Dslash library (include/coarse_dslash.h): argument
// validation, object lifetimes, halo layout, autotuning + tune cache, apply dispatch.
//
// Every entry point catches everything: no C++ exception crosses the ABI; failures return a
// cd_status and set a thread-local message (cd_last_error).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <memory>
#include <string>
#include <vector>

#include "cd_internal.h"
#include "comm.h"

namespace cd {
cudaError_t launch_dslash_f32_24(int, const ApplyArgs &, cudaStream_t, bool, int);
cudaError_t launch_dslash_f32_32(int, const ApplyArgs &, cudaStream_t, bool, int);
cudaError_t launch_dslash_f16_24(int, const ApplyArgs &, cudaStream_t, bool, int);
cudaError_t launch_dslash_f16_32(int, const ApplyArgs &, cudaStream_t, bool, int);
cudaError_t launch_halo_f32_24(const ApplyArgs &, cudaStream_t);
cudaError_t launch_halo_f32_32(const ApplyArgs &, cudaStream_t);
cudaError_t launch_halo_f16_24(const ApplyArgs &, cudaStream_t);
cudaError_t launch_halo_f16_32(const ApplyArgs &, cudaStream_t);
cudaError_t launch_pack_f32_24(const void *, const PackDst &, const KGeom &, cudaStream_t);
cudaError_t launch_pack_f32_32(const void *, const PackDst &, const KGeom &, cudaStream_t);
cudaError_t launch_pack_f16_24(const void *, const PackDst &, const KGeom &, cudaStream_t);
cudaError_t launch_pack_f16_32(const void *, const PackDst &, const KGeom &, cudaStream_t);
int variant_count_f32_24();
int variant_count_f32_32();
int variant_count_f16_24();
int variant_count_f16_32();
const char *variant_name_f32_24(int);
const char *variant_name_f32_32(int);
const char *variant_name_f16_24(int);
const char *variant_name_f16_32(int);
int variant_kind_f32_24(int, int *, int *);
int variant_kind_f32_32(int, int *, int *);
int variant_kind_f16_24(int, int *, int *);
int variant_kind_f16_32(int, int *, int *);

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches += (uint64_t)n; }

#define PICK(p, nv, f32_24, f32_32, f16_24, f16_32) \
    ((p) == CD_FP32 ? ((nv) == 24 ? (f32_24) : (f32_32)) : ((nv) == 24 ? (f16_24) : (f16_32)))

int variant_count(cd_precision p, int nv)
{
    return PICK(p, nv, variant_count_f32_24(), variant_count_f32_32(), variant_count_f16_24(), variant_count_f16_32());
}
const char *variant_name(cd_precision p, int nv, int id)
{
    return PICK(p, nv, variant_name_f32_24(id), variant_name_f32_32(id), variant_name_f16_24(id),
                variant_name_f16_32(id));
}
static int variant_kind(cd_precision p, int nv, int id, int *kw, int *wr)
{
    return PICK(p, nv, variant_kind_f32_24(id, kw, wr), variant_kind_f32_32(id, kw, wr),
                variant_kind_f16_24(id, kw, wr), variant_kind_f16_32(id, kw, wr));
}
bool variant_valid(cd_precision p, int nv, int id, const KGeom &) { return id >= 0 && id < variant_count(p, nv); }

// Heuristic when tuning is off (or the stream is being captured before a key was tuned):
// the persistent TMA ring once there are several sites per SM, else the fine-grained kernel
// with the most CTAs per site that still keeps warps busy.
int variant_heuristic(cd_precision p, int nv, const KGeom &g, int num_sms)
{
    if (g.V >= 4 * num_sms) return 0;
    int best = -1, best_score = -1;
    for (int id = 0; id < variant_count(p, nv); id++) {
        int kw = 0, wr = 0;
        if (variant_kind(p, nv, id, &kw, &wr) != 1) continue;
        const int R = (p == CD_FP32) ? 4 : 8;
        const int nrb = 2 * nv / (wr * R);
        const int64_t ctas = (int64_t)g.V * nrb;
        // prefer >= 2 CTAs per SM, then fewer hops per warp (shorter dependent chains)
        const int score = (ctas >= 2 * num_sms ? 1000 : (int)(ctas * 500 / (2 * num_sms))) - kw * 10 + wr;
        if (score > best_score) best_score = score, best = id;
    }
    return best < 0 ? 0 : best;
}

cudaError_t launch_dslash(cd_precision p, int id, const ApplyArgs &a, cudaStream_t s, bool pdl, int sms)
{
    return PICK(p, a.nvec, launch_dslash_f32_24(id, a, s, pdl, sms), launch_dslash_f32_32(id, a, s, pdl, sms),
                launch_dslash_f16_24(id, a, s, pdl, sms), launch_dslash_f16_32(id, a, s, pdl, sms));
}
cudaError_t launch_halo(cd_precision p, const ApplyArgs &a, cudaStream_t s)
{
    return PICK(p, a.nvec, launch_halo_f32_24(a, s), launch_halo_f32_32(a, s), launch_halo_f16_24(a, s),
                launch_halo_f16_32(a, s));
}
cudaError_t launch_chain_f32_24(int, const ApplyArgs &, int, unsigned, cudaStream_t, int, int *);
cudaError_t launch_chain_f32_32(int, const ApplyArgs &, int, unsigned, cudaStream_t, int, int *);
cudaError_t launch_chain_f16_24(int, const ApplyArgs &, int, unsigned, cudaStream_t, int, int *);
cudaError_t launch_chain_f16_32(int, const ApplyArgs &, int, unsigned, cudaStream_t, int, int *);
cudaError_t launch_chain(cd_precision p, int id, const ApplyArgs &a, int n, unsigned base, cudaStream_t s, int sms,
                         int *nrb)
{
    return PICK(p, a.nvec, launch_chain_f32_24(id, a, n, base, s, sms, nrb),
                launch_chain_f32_32(id, a, n, base, s, sms, nrb), launch_chain_f16_24(id, a, n, base, s, sms, nrb),
                launch_chain_f16_32(id, a, n, base, s, sms, nrb));
}
cudaError_t launch_ringh_f32_24(const ApplyArgs &, cudaStream_t, bool, int, int);
cudaError_t launch_ringh_f32_32(const ApplyArgs &, cudaStream_t, bool, int, int);
cudaError_t launch_ringh_f16_24(const ApplyArgs &, cudaStream_t, bool, int, int);
cudaError_t launch_ringh_f16_32(const ApplyArgs &, cudaStream_t, bool, int, int);
cudaError_t launch_ringh(cd_precision p, const ApplyArgs &a, cudaStream_t s, bool pdl, int sms, int mps)
{
    return PICK(p, a.nvec, launch_ringh_f32_24(a, s, pdl, sms, mps), launch_ringh_f32_32(a, s, pdl, sms, mps),
                launch_ringh_f16_24(a, s, pdl, sms, mps), launch_ringh_f16_32(a, s, pdl, sms, mps));
}
cudaError_t launch_fgh_f32_24(const ApplyArgs &, cudaStream_t, bool);
cudaError_t launch_fgh_f32_32(const ApplyArgs &, cudaStream_t, bool);
cudaError_t launch_fgh_f16_24(const ApplyArgs &, cudaStream_t, bool);
cudaError_t launch_fgh_f16_32(const ApplyArgs &, cudaStream_t, bool);
cudaError_t launch_compress_f32_24(const void *, void *, int64_t, cudaStream_t);
cudaError_t launch_compress_f32_32(const void *, void *, int64_t, cudaStream_t);
cudaError_t launch_compress_f16_24(const void *, void *, int64_t, cudaStream_t);
cudaError_t launch_compress_f16_32(const void *, void *, int64_t, cudaStream_t);
cudaError_t launch_hermdev_f32_24(const void *, const KGeom &, float *, cudaStream_t, const void *, const int64_t *);
cudaError_t launch_hermdev_f32_32(const void *, const KGeom &, float *, cudaStream_t, const void *, const int64_t *);
cudaError_t launch_hermdev_f16_24(const void *, const KGeom &, float *, cudaStream_t, const void *, const int64_t *);
cudaError_t launch_hermdev_f16_32(const void *, const KGeom &, float *, cudaStream_t, const void *, const int64_t *);
cudaError_t launch_fgh_halo_f32_24(const ApplyArgs &, cudaStream_t);
cudaError_t launch_fgh_halo_f32_32(const ApplyArgs &, cudaStream_t);
cudaError_t launch_fgh_halo_f16_24(const ApplyArgs &, cudaStream_t);
cudaError_t launch_fgh_halo_f16_32(const ApplyArgs &, cudaStream_t);
cudaError_t launch_lhalo_pack_f32_24(const void *, void *, const KGeom &, const int64_t *, cudaStream_t);
cudaError_t launch_lhalo_pack_f32_32(const void *, void *, const KGeom &, const int64_t *, cudaStream_t);
cudaError_t launch_lhalo_pack_f16_24(const void *, void *, const KGeom &, const int64_t *, cudaStream_t);
cudaError_t launch_lhalo_pack_f16_32(const void *, void *, const KGeom &, const int64_t *, cudaStream_t);
cudaError_t launch_fgh_halo(cd_precision p, const ApplyArgs &a, cudaStream_t s)
{
    return PICK(p, a.nvec, launch_fgh_halo_f32_24(a, s), launch_fgh_halo_f32_32(a, s), launch_fgh_halo_f16_24(a, s),
                launch_fgh_halo_f16_32(a, s));
}
cudaError_t launch_lhalo_pack(cd_precision p, int nv, const void *c, void *d, const KGeom &g, const int64_t *o,
                              cudaStream_t s)
{
    return PICK(p, nv, launch_lhalo_pack_f32_24(c, d, g, o, s), launch_lhalo_pack_f32_32(c, d, g, o, s),
                launch_lhalo_pack_f16_24(c, d, g, o, s), launch_lhalo_pack_f16_32(c, d, g, o, s));
}
cudaError_t launch_fgh(cd_precision p, const ApplyArgs &a, cudaStream_t s, bool pdl)
{
    return PICK(p, a.nvec, launch_fgh_f32_24(a, s, pdl), launch_fgh_f32_32(a, s, pdl), launch_fgh_f16_24(a, s, pdl),
                launch_fgh_f16_32(a, s, pdl));
}
cudaError_t launch_compress(cd_precision p, int nv, const void *f, void *c, int64_t n, cudaStream_t s)
{
    return PICK(p, nv, launch_compress_f32_24(f, c, n, s), launch_compress_f32_32(f, c, n, s),
                launch_compress_f16_24(f, c, n, s), launch_compress_f16_32(f, c, n, s));
}
cudaError_t launch_hermdev(cd_precision p, int nv, const void *f, const KGeom &g, float *d, cudaStream_t s,
                           const void *lh, const int64_t *lo)
{
    return PICK(p, nv, launch_hermdev_f32_24(f, g, d, s, lh, lo), launch_hermdev_f32_32(f, g, d, s, lh, lo),
                launch_hermdev_f16_24(f, g, d, s, lh, lo), launch_hermdev_f16_32(f, g, d, s, lh, lo));
}
cudaError_t launch_pack(cd_precision p, int nv, const void *f, const PackDst &d, const KGeom &g, cudaStream_t s)
{
    return PICK(p, nv, launch_pack_f32_24(f, d, g, s), launch_pack_f32_32(f, d, g, s), launch_pack_f16_24(f, d, g, s),
                launch_pack_f16_32(f, d, g, s));
}

}  // namespace cd

using namespace cd;

// ------------------------------------------------------------------ errors
static thread_local std::string t_err;

static int fail(int code, const std::string &msg)
{
    t_err = msg;
    return code;
}
static int cuda_fail(cudaError_t e, const char *what)
{
    return fail(CD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_TRY(expr, what)                         \
    do {                                             \
        cudaError_t e_ = (expr);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

#define API_BEGIN try {
#define API_END                                                          \
    }                                                                    \
    catch (const std::exception &ex) { return fail(CD_ERR_INVALID, ex.what()); } \
    catch (...) { return fail(CD_ERR_INVALID, "unknown C++ exception"); }

static cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }
static int64_t field_sites(const cd_field *f) { return f->parity < 0 ? f->ctx->V : f->ctx->V / 2; }

// Device allocation owned until release(): early error returns free it (cudaFree synchronises
// the device, which is fine on these setup-time error paths).
struct DevBuf {
    void *p = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf()
    {
        if (p) cudaFree(p);
    }
    void *release()
    {
        void *q = p;
        p = nullptr;
        return q;
    }
};

// Makes the context's device current for the duration of an entry point and restores the
// caller's device afterwards (a process may hold contexts on several GPUs).
struct DevGuard {
    int prev = -1;
    bool changed = false;
    explicit DevGuard(int dev)
    {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) changed = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DevGuard()
    {
        if (changed) cudaSetDevice(prev);
    }
    DevGuard(const DevGuard &) = delete;
    DevGuard &operator=(const DevGuard &) = delete;
};
#define CTX_GUARD(ctx) DevGuard dev_guard_((ctx)->device)

// ------------------------------------------------------------------ decomposition + halo plan
// Geometry checks shared by cd_context_create and cd_halo_plan_create.
static int check_geometry(const cd_geometry *geom, int nranks, int rank)
{
    if (!geom) return fail(CD_ERR_INVALID, "geom is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CD_ERR_INVALID, "bad nranks/rank");
    int64_t prodP = 1, V = 1;
    for (int mu = 0; mu < 4; mu++) {
        if (geom->global_dims[mu] < 1) return fail(CD_ERR_INVALID, "global_dims must be >= 1");
        if (geom->proc_grid[mu] < 1) return fail(CD_ERR_INVALID, "proc_grid must be >= 1");
        if (geom->global_dims[mu] % geom->proc_grid[mu]) return fail(CD_ERR_INVALID, "global_dims % proc_grid != 0");
        prodP *= geom->proc_grid[mu];
        V *= geom->global_dims[mu] / geom->proc_grid[mu];
    }
    if (prodP != nranks) return fail(CD_ERR_INVALID, "prod(proc_grid) != nranks");
    if (geom->nvec != 24 && geom->nvec != 32) return fail(CD_ERR_UNSUPPORTED, "nvec must be 24 or 32");
    if (V >= (int64_t(1) << 31) / 9) return fail(CD_ERR_UNSUPPORTED, "local volume too large");
    return CD_OK;
}

// Rank grid (lexicographic like sites), local block, periodic neighbour ranks, and the wire
// layout of DESIGN.md R13: split dims ascending; per dim block A (face sent to +mu, x_mu =
// L-1) then block B (face sent to -mu, x_mu = 0); each block = F payload records then (fp16)
// F float scales, zero-padded to 16 bytes.
static void make_plan(const cd_geometry *geom, int rank, cd_precision p, int self_mask, cd_halo_plan *o)
{
    memset(o, 0, sizeof(*o));
    const int N = 2 * geom->nvec;
    int t = rank;
    o->local_volume = 1;
    for (int mu = 0; mu < 4; mu++) {
        o->grid_coords[mu] = t % geom->proc_grid[mu];
        t /= geom->proc_grid[mu];
        o->local_dims[mu] = geom->global_dims[mu] / geom->proc_grid[mu];
        o->local_volume *= o->local_dims[mu];
        if (geom->proc_grid[mu] > 1 || ((self_mask >> mu) & 1)) o->split_mask |= 1 << mu;
    }
    for (int mu = 0; mu < 4; mu++)
        for (int dir = 0; dir < 2; dir++) {
            int cc[4] = {o->grid_coords[0], o->grid_coords[1], o->grid_coords[2], o->grid_coords[3]};
            const int P = geom->proc_grid[mu];
            cc[mu] = (cc[mu] + (dir == 0 ? 1 : -1) + P) % P;
            o->nbr_rank[mu][dir] = ((cc[3] * geom->proc_grid[2] + cc[2]) * geom->proc_grid[1] + cc[1]) *
                                       geom->proc_grid[0] + cc[0];
        }
    o->record_bytes = (p == CD_FP32) ? 8 * (int64_t)N : 4 * (int64_t)N;
    o->scale_bytes = (p == CD_FP32) ? 0 : 4;
    int64_t off = 0;
    for (int mu = 0; mu < 4; mu++) {
        o->face_sites[mu] = o->local_volume / o->local_dims[mu];
        if (!((o->split_mask >> mu) & 1)) continue;
        o->block_bytes[mu] = (o->face_sites[mu] * (o->record_bytes + o->scale_bytes) + 15) & ~int64_t(15);
        for (int b = 0; b < 2; b++) {
            o->block_offset[mu][b] = off;
            off += o->block_bytes[mu];
        }
    }
    o->total_bytes = off;
}

static cd_halo_plan ctx_plan(const cd_context *c, cd_precision p)
{
    cd_halo_plan o;
    make_plan(&c->geom, c->rank, p, c->halo_self_mask, &o);
    return o;
}

static KGeom halo_geom(const cd_context *c, cd_precision p)
{
    KGeom g = c->kg;
    const cd_halo_plan pl = ctx_plan(c, p);
    for (int mu = 0; mu < 4; mu++) {
        g.F[mu] = (int)pl.face_sites[mu];
        g.blk_off[mu][0] = pl.block_offset[mu][0];
        g.blk_off[mu][1] = pl.block_offset[mu][1];
    }
    return g;
}
static size_t halo_bytes(const cd_context *c, cd_precision p) { return (size_t)ctx_plan(c, p).total_bytes; }

static int setup_halo(cd_context *c)
{
    if (c->halo_ready || c->kg.split == 0) return CD_OK;
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t cap = align256(std::max(halo_bytes(c, CD_FP32), halo_bytes(c, CD_FP16)) + 16);
    CUDA_TRY(cudaMalloc(&c->send_buf, cap), "cudaMalloc(send)");
    CUDA_TRY(cudaMalloc(&c->recv_buf, cap), "cudaMalloc(recv)");
    CUDA_TRY(cudaMemset(c->send_buf, 0, cap), "memset");
    CUDA_TRY(cudaMemset(c->recv_buf, 0, cap), "memset");
    c->halo_cap = cap;
    CUDA_TRY(cudaMalloc(&c->face_scratch, sizeof(float2) * c->V * c->N), "cudaMalloc(scratch)");
    std::vector<int> faces, interior;
    for (int64_t s = 0; s < c->V; s++) {
        int64_t t = s;
        int x[4];
        for (int mu = 0; mu < 4; mu++) {
            x[mu] = (int)(t % c->local[mu]);
            t /= c->local[mu];
        }
        bool face = false;
        for (int mu = 0; mu < 4; mu++)
            if (((c->kg.split >> mu) & 1) && (x[mu] == 0 || x[mu] == c->local[mu] - 1)) face = true;
        if (face) faces.push_back((int)s);
        else interior.push_back((int)s);
    }
    c->n_face = (int)faces.size();
    c->n_interior = (int)interior.size();
    CUDA_TRY(cudaMalloc(&c->interior_sites, sizeof(int) * std::max<size_t>(1, interior.size())), "cudaMalloc(interior)");
    if (!interior.empty())
        CUDA_TRY(cudaMemcpy(c->interior_sites, interior.data(), sizeof(int) * interior.size(), cudaMemcpyHostToDevice),
                 "cudaMemcpy(interior)");
    CUDA_TRY(cudaMalloc(&c->face_sites, sizeof(int) * std::max<size_t>(1, faces.size())), "cudaMalloc(faces)");
    if (!faces.empty())
        CUDA_TRY(cudaMemcpy(c->face_sites, faces.data(), sizeof(int) * faces.size(), cudaMemcpyHostToDevice),
                 "cudaMemcpy(faces)");
    if (!c->comm_stream) {   // highest priority: the pack (+ peer put) is dispatched ahead of the interior
        int lo = 0, hi = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
        CUDA_TRY(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi), "stream");
    }
    if (!c->ev_in) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming), "event");
    if (!c->ev_halo) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming), "event");
    c->halo_ready = true;
    return CD_OK;
}

// ------------------------------------------------------------------ tune cache (file)
static std::string tune_key_str(const cd_context *c, int prec, int dag)
{
    std::ostringstream o;
    o << "v1 nvec=" << c->nvec << " prec=" << prec << " dag=" << dag << " L=" << c->local[0] << "," << c->local[1]
      << "," << c->local[2] << "," << c->local[3] << " split=" << c->kg.split << " sms=" << c->num_sms;
    return o.str();
}
static std::mutex g_tune_mu;
static int tune_file_lookup(const std::string &key)
{
    const char *path = getenv("CD_TUNE_CACHE");
    if (!path || !*path) return -1;
    std::lock_guard<std::mutex> lk(g_tune_mu);
    std::ifstream f(path);
    std::string line;
    int found = -1;
    while (std::getline(f, line)) {
        const size_t bar = line.find(" | ");
        if (bar != std::string::npos && line.substr(0, bar) == key) found = atoi(line.c_str() + bar + 3);
    }
    return found;
}
static void tune_file_store(const std::string &key, int id, const char *name, float us)
{
    const char *path = getenv("CD_TUNE_CACHE");
    if (!path || !*path) return;
    std::lock_guard<std::mutex> lk(g_tune_mu);
    std::ofstream f(path, std::ios::app);
    f << key << " | " << id << " | " << (name ? name : "?") << " | " << us << " us\n";
}

// ------------------------------------------------------------------ context
// Frees everything a (possibly half-built) context holds, then the context itself.
static void ctx_release(cd_context *c)
{
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    void *bufs[] = {c->send_buf, c->recv_buf, c->face_scratch, c->face_sites, c->interior_sites, c->mrhs_send,
                    c->mrhs_recv, c->work, c->ysplit, c->site_cnt, c->chain_cnt, c->llbuf, c->pack_cnt};
    for (void *b : bufs)
        if (b) cudaFree(b);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    peer_release(c);
    if (c->err_host) cudaFreeHost(c->err_host);
    comm_destroy(c->comm);
    delete c;
}

extern "C" {

const char *cd_version(void) { return "coarse_dslash 0.1 (sm_100a)"; }
const char *cd_last_error(void) { return t_err.c_str(); }
uint64_t cd_launch_count(void) { return g_launches.load(); }

int cd_get_unique_id(uint8_t out_id[128])
{
    API_BEGIN
    if (!out_id) return fail(CD_ERR_INVALID, "out_id is NULL");
    std::string err;
    int r = nccl_unique_id(out_id, err);
    if (r != CD_OK) return fail(r, err);
    return CD_OK;
    API_END
}

int cd_context_create(const cd_geometry *geom, int device, int nranks, int rank, const uint8_t *nccl_id,
                      cd_context **out)
{
    API_BEGIN
    if (!geom || !out) return fail(CD_ERR_INVALID, "geom/out is NULL");
    *out = nullptr;
    int r0 = check_geometry(geom, nranks, rank);
    if (r0 != CD_OK) return r0;
    if (nranks == 1 && nccl_id != nullptr) return fail(CD_ERR_INVALID, "nccl_id must be NULL for nranks == 1");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(CD_ERR_INVALID, "bad device");
    DevGuard dev_guard_(device);

    cd_context *c = new cd_context();
    c->geom = *geom;
    c->device = device;
    c->nranks = nranks;
    c->rank = rank;
    c->nvec = geom->nvec;
    c->N = 2 * geom->nvec;
    cd_halo_plan pl;
    make_plan(geom, rank, CD_FP32, 0, &pl);
    for (int mu = 0; mu < 4; mu++) {
        c->coords[mu] = pl.grid_coords[mu];
        c->local[mu] = pl.local_dims[mu];
        c->nbr_rank[mu][0] = pl.nbr_rank[mu][0];
        c->nbr_rank[mu][1] = pl.nbr_rank[mu][1];
    }
    c->V = pl.local_volume;
    KGeom &g = c->kg;
    for (int mu = 0; mu < 4; mu++) g.L[mu] = c->local[mu];
    g.V = (int)c->V;
    for (int i = 0; i < 3; i++) g.fd[i] = make_fastdiv((uint32_t)c->local[i]);
    g.split = pl.split_mask;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        ctx_release(c);
        return cuda_fail(e, "cudaGetDeviceProperties");
    }
    c->num_sms = prop.multiProcessorCount;
    e = cudaMalloc(&c->work, 8 * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->work, 0, 8 * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->ysplit, sizeof(float2) * c->V * c->N);
    if (e == cudaSuccess) e = cudaMalloc(&c->site_cnt, sizeof(int) * c->V);
    if (e == cudaSuccess) e = cudaMemset(c->site_cnt, 0, sizeof(int) * c->V);
    if (e == cudaSuccess) {   // host-mapped transport error word (in-kernel arrival-wait timeouts)
        e = cudaHostAlloc(reinterpret_cast<void **>(&c->err_host), sizeof(int), cudaHostAllocMapped);
        if (e == cudaSuccess) {
            *c->err_host = 0;
            e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->err_dev), c->err_host, 0);
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->pack_cnt, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->pack_cnt, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->chain_cnt, sizeof(unsigned) * c->V);
    if (e == cudaSuccess) e = cudaMemset(c->chain_cnt, 0, sizeof(unsigned) * c->V);
    if (e != cudaSuccess) {
        ctx_release(c);
        return cuda_fail(e, "cudaMalloc(work)");
    }
    if (const char *ev = getenv("CD_TUNE")) c->tune = atoi(ev) ? 1 : 0;
    if (const char *ev = getenv("CD_VARIANT")) c->force_variant = atoi(ev);
    if (const char *ev = getenv("CD_PDL")) c->pdl = atoi(ev) ? 1 : 0;
    if (const char *ev = getenv("CD_FUSE_SPLIT")) c->fuse_split = atoi(ev) ? 1 : 0;
    if (nranks > 1 && nccl_id) {
        std::string err;
        int r = comm_create(nccl_id, nranks, rank, &c->comm, err);
        if (r != CD_OK) {
            ctx_release(c);
            return fail(r, err);
        }
    }
    int r = setup_halo(c);
    if (r != CD_OK) {
        ctx_release(c);
        return r;
    }
    *out = c;
    return CD_OK;
    API_END
}

int cd_context_destroy(cd_context *c)
{
    API_BEGIN
    if (!c) return fail(CD_ERR_INVALID, "ctx is NULL");
    DevGuard dev_guard_(c->device);
    ctx_release(c);
    return CD_OK;
    API_END
}

int cd_context_set_option(cd_context *c, int option, int64_t value)
{
    API_BEGIN
    if (!c) return fail(CD_ERR_INVALID, "ctx is NULL");
    CTX_GUARD(c);
    std::lock_guard<std::mutex> lk(c->mu);
    switch (option) {
    case CD_OPT_VARIANT:
        if (value < -1) return fail(CD_ERR_INVALID, "variant must be >= -1");
        c->force_variant = (int)value;
        return CD_OK;
    case CD_OPT_TUNE:
        c->tune = value ? 1 : 0;
        return CD_OK;
    case CD_OPT_PDL:
        c->pdl = value ? 1 : 0;
        return CD_OK;
    case CD_OPT_TRANSPORT: {
        if (value < TR_AUTO || value > TR_COPY) return fail(CD_ERR_INVALID, "transport must be 0 (auto), 1 (NCCL), 2 (peer), 3 (copy)");
        if (value == TR_NCCL && !c->comm) {
            if (c->nranks != 1)
                return fail(CD_ERR_INVALID, "NCCL transport on a multi-rank context needs the nccl_id at creation");
            std::string err;
            int r = comm_create_self(&c->comm, err);   // 1 rank: the halo self exchanges go through NCCL
            if (r != CD_OK) return fail(r, err);
        }
        if (value == TR_PEER && !c->peer_ready)
            return fail(CD_ERR_INVALID, "peer transport needs cd_context_peer_handle + cd_context_peer_connect first");
        if (value == TR_COPY && c->nranks != 1) return fail(CD_ERR_INVALID, "device-copy transport is single-rank");
        c->transport = (int)value;
        c->chosen.clear();   // the interior's SM budget depends on the transport
        return CD_OK;
    }
    case CD_OPT_NCCL_SM_RESERVE:
        if (value < 0 || value >= c->num_sms) return fail(CD_ERR_INVALID, "SM reserve must be in [0, num_sms)");
        c->nccl_sm_reserve = (int)value;
        c->chosen.clear();
        return CD_OK;
    case CD_OPT_PEER_TIMEOUT_MS:
        if (value < 1) return fail(CD_ERR_INVALID, "timeout must be >= 1 ms");
        c->peer_timeout_ns = (unsigned long long)value * 1000000ull;
        return CD_OK;
    case CD_OPT_HALO_SELF_MASK: {
        if (value < 0 || value > 15) return fail(CD_ERR_INVALID, "mask must be in [0, 15]");
        if (c->applied) return fail(CD_ERR_INVALID, "HALO_SELF_MASK must be set before the first apply");
        if (c->win) return fail(CD_ERR_INVALID, "HALO_SELF_MASK must be set before cd_context_peer_handle");
        for (int mu = 0; mu < 4; mu++)
            if (((value >> mu) & 1) && c->geom.proc_grid[mu] != 1)
                return fail(CD_ERR_INVALID, "HALO_SELF_MASK dims must have proc_grid == 1");
        if (c->halo_ready) {
            cudaFree(c->send_buf);
            cudaFree(c->recv_buf);
            cudaFree(c->face_scratch);
            cudaFree(c->face_sites);
            cudaFree(c->interior_sites);
            if (c->mrhs_send) cudaFree(c->mrhs_send);
            if (c->mrhs_recv) cudaFree(c->mrhs_recv);
            c->send_buf = c->recv_buf = nullptr;
            c->face_scratch = nullptr;
            c->face_sites = nullptr;
            c->interior_sites = nullptr;
            c->mrhs_send = c->mrhs_recv = nullptr;
            c->mrhs_cap = 0;
            c->halo_ready = false;
        }
        c->halo_self_mask = (int)value;
        int split = 0;
        for (int mu = 0; mu < 4; mu++)
            if (c->geom.proc_grid[mu] > 1) split |= (1 << mu);
        c->kg.split = split | (int)value;
        c->chosen.clear();
        return setup_halo(c);
    }
    default:
        return fail(CD_ERR_INVALID, "unknown option");
    }
    API_END
}

int cd_context_local(const cd_context *c, int32_t local_dims[4], int64_t *local_volume, int32_t grid_coords[4])
{
    if (!c) return fail(CD_ERR_INVALID, "ctx is NULL");
    for (int mu = 0; mu < 4; mu++) {
        if (local_dims) local_dims[mu] = c->local[mu];
        if (grid_coords) grid_coords[mu] = c->coords[mu];
    }
    if (local_volume) *local_volume = c->V;
    return CD_OK;
}

int cd_variant_count(const cd_context *c, cd_precision p)
{
    if (!c || (p != CD_FP32 && p != CD_FP16)) return 0;
    return variant_count(p, c->nvec);
}
const char *cd_variant_name(const cd_context *c, cd_precision p, int id)
{
    if (!c || (p != CD_FP32 && p != CD_FP16)) return nullptr;
    return variant_name(p, c->nvec, id);
}
int cd_context_chosen_variant(const cd_context *c, cd_precision p, int dagger)
{
    if (!c) return -1;
    auto *cc = const_cast<cd_context *>(c);
    std::lock_guard<std::mutex> lk(cc->mu);
    auto it = c->chosen.find(TuneKey{(int)p, dagger >= 2 ? (dagger & 3) : (dagger ? 1 : 0)});
    return it == c->chosen.end() ? -1 : it->second;
}

// ------------------------------------------------------------------ fields
size_t coarse_field_bytes(const cd_context *c, cd_precision p)
{
    if (!c || (p != CD_FP32 && p != CD_FP16)) return 0;
    return align256(vec_rec_bytes(c->N, p) * (size_t)c->V);
}

int coarse_field_alloc(cd_context *c, cd_precision p, void *mem, size_t bytes, cd_field **out)
{
    API_BEGIN
    if (!c || !out) return fail(CD_ERR_INVALID, "ctx/out is NULL");
    if (p != CD_FP32 && p != CD_FP16) return fail(CD_ERR_INVALID, "bad precision");
    CTX_GUARD(c);
    const size_t need = coarse_field_bytes(c, p);
    bool owned = false;
    if (!mem) {
        CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
        cudaError_t e = cudaMalloc(&mem, need);
        if (e != cudaSuccess) return fail(CD_ERR_OOM, std::string("cudaMalloc(field): ") + cudaGetErrorString(e));
        bytes = need;
        owned = true;
    } else {
        if (reinterpret_cast<uintptr_t>(mem) % 256) return fail(CD_ERR_INVALID, "device_mem must be 256-B aligned");
        if (bytes < need) return fail(CD_ERR_INVALID, "device_mem too small (need coarse_field_bytes)");
    }
    *out = new cd_field{c, p, mem, bytes, owned, 1, -1};
    return CD_OK;
    API_END
}

size_t coarse_field_bytes_mrhs(const cd_context *c, cd_precision p, int nrhs)
{
    if (!c || (p != CD_FP32 && p != CD_FP16) || nrhs < 1) return 0;
    if (p == CD_FP16 && nrhs > 1) {   // tensor-core block layout (R22): 128 rhs per block
        if (nrhs % 128) return 0;
        return align256(((size_t)128 * 4 * c->N + 16) * (size_t)c->V * (size_t)(nrhs / 128));
    }
    return align256(vec_rec_bytes(c->N, p) * (size_t)c->V * (size_t)nrhs);
}

int coarse_field_alloc_mrhs(cd_context *c, cd_precision p, int nrhs, void *mem, size_t bytes, cd_field **out)
{
    API_BEGIN
    if (!c || !out) return fail(CD_ERR_INVALID, "ctx/out is NULL");
    if (p != CD_FP32 && p != CD_FP16) return fail(CD_ERR_INVALID, "bad precision");
    if (nrhs < 1) return fail(CD_ERR_INVALID, "nrhs must be >= 1");
    CTX_GUARD(c);
    if (p == CD_FP16 && nrhs > 1 && nrhs % 128)
        return fail(CD_ERR_UNSUPPORTED, "fp16 multi-RHS fields hold blocks of 128 right-hand sides (nrhs % 128 == 0)");
    const size_t need = coarse_field_bytes_mrhs(c, p, nrhs);
    bool owned = false;
    if (!mem) {
        CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
        cudaError_t e = cudaMalloc(&mem, need);
        if (e != cudaSuccess) return fail(CD_ERR_OOM, std::string("cudaMalloc(field): ") + cudaGetErrorString(e));
        bytes = need;
        owned = true;
    } else {
        if (reinterpret_cast<uintptr_t>(mem) % 256) return fail(CD_ERR_INVALID, "device_mem must be 256-B aligned");
        if (bytes < need) return fail(CD_ERR_INVALID, "device_mem too small (need coarse_field_bytes_mrhs)");
    }
    *out = new cd_field{c, p, mem, bytes, owned, nrhs, -1};
    return CD_OK;
    API_END
}

int coarse_field_free(cd_field *f)
{
    API_BEGIN
    if (!f) return fail(CD_ERR_INVALID, "field is NULL");
    if (f->owned) cudaFree(f->base);   // cudaFree needs no current device (and f->ctx may be gone)
    delete f;
    return CD_OK;
    API_END
}

// Bounded device staging for host <-> device transfers of canonical data.
static int staged_h2d(void *dst_dev, const void *src_host, size_t bytes, cudaStream_t s)
{
    CUDA_TRY(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D)");
    return CD_OK;
}

int coarse_field_import(cd_field *f, const void *src, int src_on_device, cd_host_dtype dt, void *stream)
{
    API_BEGIN
    if (!f || !src) return fail(CD_ERR_INVALID, "field/src is NULL");
    if (dt != CD_C64 && dt != CD_C128) return fail(CD_ERR_INVALID, "bad dtype");
    CTX_GUARD(f->ctx);
    cd_context *c = f->ctx;
    const size_t elem = dt == CD_C128 ? 16 : 8;
    const size_t bytes = elem * c->N * (size_t)field_sites(f) * f->nrhs;
    cudaStream_t s = S(stream);
    if (f->prec == CD_FP32 && dt == CD_C64 && f->nrhs == 1) {   // stored layout == canonical layout
        CUDA_TRY(cudaMemcpyAsync(f->base, src, bytes, src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 s), "cudaMemcpyAsync(import)");
        return CD_OK;
    }
    const void *dsrc = src;
    void *stage = nullptr;
    if (!src_on_device) {
        CUDA_TRY(cudaMallocAsync(&stage, bytes, s), "cudaMallocAsync(stage)");
        int r = staged_h2d(stage, src, bytes, s);
        if (r != CD_OK) return r;
        dsrc = stage;
    }
    CUDA_TRY(launch_import(f->prec, c->nvec, field_sites(f), dsrc, dt == CD_C128, f->base, s, f->nrhs), "import kernel");
    if (stage) CUDA_TRY(cudaFreeAsync(stage, s), "cudaFreeAsync");
    return CD_OK;
    API_END
}

int coarse_field_export(const cd_field *f, void *dst, int dst_on_device, cd_host_dtype dt, void *stream)
{
    API_BEGIN
    if (!f || !dst) return fail(CD_ERR_INVALID, "field/dst is NULL");
    if (dt != CD_C64 && dt != CD_C128) return fail(CD_ERR_INVALID, "bad dtype");
    CTX_GUARD(f->ctx);
    cd_context *c = f->ctx;
    const size_t elem = dt == CD_C128 ? 16 : 8;
    const size_t bytes = elem * c->N * (size_t)field_sites(f) * f->nrhs;
    cudaStream_t s = S(stream);
    if (f->prec == CD_FP32 && dt == CD_C64 && f->nrhs == 1) {
        CUDA_TRY(cudaMemcpyAsync(dst, f->base, bytes, dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 s), "cudaMemcpyAsync(export)");
        return CD_OK;
    }
    void *ddst = dst;
    void *stage = nullptr;
    if (!dst_on_device) {
        CUDA_TRY(cudaMallocAsync(&stage, bytes, s), "cudaMallocAsync(stage)");
        ddst = stage;
    }
    CUDA_TRY(launch_export(f->prec, c->nvec, field_sites(f), f->base, ddst, dt == CD_C128, s, f->nrhs), "export kernel");
    if (stage) {
        CUDA_TRY(cudaMemcpyAsync(dst, stage, bytes, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(D2H)");
        CUDA_TRY(cudaFreeAsync(stage, s), "cudaFreeAsync");
    }
    return CD_OK;
    API_END
}

int coarse_field_generate(cd_field *f, uint64_t seed, uint32_t tag, int32_t scale_log2, void *stream)
{
    API_BEGIN
    if (!f) return fail(CD_ERR_INVALID, "field is NULL");
    CTX_GUARD(f->ctx);
    if (scale_log2 < -60 || scale_log2 > 60) return fail(CD_ERR_INVALID, "scale_log2 out of range");
    if (f->parity >= 0) return fail(CD_ERR_UNSUPPORTED, "generate: full-lattice fields only");
    CUDA_TRY(launch_field_generate(f->prec, f->ctx->nvec, f->ctx, seed, tag, scale_log2, f->base, S(stream), f->nrhs),
             "field generate");
    return CD_OK;
    API_END
}

size_t coarse_field_stored_bytes(const cd_field *f)
{
    if (!f) return 0;
    const size_t recs = (size_t)field_sites(f) * f->nrhs;
    const size_t n = recs * f->ctx->N;
    if (f->prec == CD_FP16 && f->nrhs > 1) return (size_t)field_sites(f) * (f->nrhs / 128) * (128 * 4 * f->ctx->N + 16);
    return f->prec == CD_FP32 ? 8 * n : 4 * n + 4 * recs;
}

// internal records -> canonical raw (payloads contiguous, then scales), via the host
static int read_stored(const void *base, int64_t nrec, size_t payload, size_t rec, bool f16, void *dst,
                       int dst_on_device, cudaStream_t s)
{
    std::vector<unsigned char> h(rec * nrec);
    CUDA_TRY(cudaMemcpyAsync(h.data(), base, h.size(), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(read)");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    std::vector<unsigned char> o(payload * nrec + (f16 ? 4 * nrec : 0));
    for (int64_t r = 0; r < nrec; r++) {
        memcpy(o.data() + payload * r, h.data() + rec * r, payload);
        if (f16) memcpy(o.data() + payload * nrec + 4 * r, h.data() + rec * r + payload, 4);
    }
    if (dst_on_device) {
        CUDA_TRY(cudaMemcpy(dst, o.data(), o.size(), cudaMemcpyHostToDevice), "cudaMemcpy(read)");
    } else {
        memcpy(dst, o.data(), o.size());
    }
    return CD_OK;
}

int coarse_field_read_stored(const cd_field *f, void *dst, int dst_on_device, void *stream)
{
    API_BEGIN
    if (!f || !dst) return fail(CD_ERR_INVALID, "field/dst is NULL");
    CTX_GUARD(f->ctx);
    const int N = f->ctx->N;
    const bool f16 = f->prec == CD_FP16;
    if (f16 && f->nrhs > 1) {   // tensor-core blocks are returned as stored (R22)
        const size_t n = coarse_field_stored_bytes(f);
        CUDA_TRY(cudaMemcpyAsync(dst, f->base, n, dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 S(stream)),
                 "cudaMemcpyAsync(read)");
        CUDA_TRY(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize");
        return CD_OK;
    }
    return read_stored(f->base, field_sites(f) * f->nrhs, f16 ? 4 * N : 8 * N, vec_rec_bytes(N, f->prec), f16, dst, dst_on_device,
                       S(stream));
    API_END
}

// ------------------------------------------------------------------ links
static int links_new(cd_context *c, cd_precision p, cd_links **out, int compressed = 0)
{
    const size_t bytes = align256(mat_rec_bytes(c->N, p) * (compressed ? 5 : 9) * (size_t)c->V);
    void *mem = nullptr;
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    cudaError_t e = cudaMalloc(&mem, bytes);
    if (e != cudaSuccess) return fail(CD_ERR_OOM, std::string("cudaMalloc(links): ") + cudaGetErrorString(e));
    *out = new cd_links{c, p, mem, bytes, compressed, 0, nullptr, nullptr};
    return CD_OK;
}

int coarse_links_compress_hermitian(const cd_links *full, double *max_dev, void *stream, cd_links **out)
{
    API_BEGIN
    if (!full || !out) return fail(CD_ERR_INVALID, "links/out is NULL");
    CTX_GUARD(full->ctx);
    if (full->compressed) return fail(CD_ERR_INVALID, "links are already compressed");
    if (full->eo) return fail(CD_ERR_INVALID, "even-odd prepared links cannot be compressed");
    cd_context *c = full->ctx;
    cudaStream_t s = S(stream);
    cd_links *l = nullptr;
    int r = links_new(c, full->prec, &l, 1);
    if (r != CD_OK) return r;
    std::unique_ptr<cd_links, int (*)(cd_links *)> guard(l, coarse_links_free);
    l->split = c->kg.split;
    CUDA_TRY(launch_compress(full->prec, c->nvec, full->base, l->base, c->V, s), "links compress");
    if (c->kg.split != 0) {
        // multi-rank: a ONE-TIME link halo -- the backward hop of an x_mu = 0 site needs the -mu
        // neighbour rank's forward record L_{2mu}(x - mu); every rank sends its x_mu = L-1 face
        // records to the +mu neighbour (block A of the exchange; block B is unused).
        const size_t mrec = mat_rec_bytes(c->N, full->prec);
        cd_halo_plan pl = ctx_plan(c, full->prec);
        int64_t off = 0;
        for (int mu = 0; mu < 4; mu++) {
            pl.block_offset[mu][0] = pl.block_offset[mu][1] = 0;
            pl.block_bytes[mu] = 0;
            if (!((c->kg.split >> mu) & 1)) continue;
            const int64_t b = (int64_t)(c->V / c->local[mu]) * (int64_t)mrec;
            pl.block_offset[mu][0] = l->lhoff[mu] = off;
            pl.block_offset[mu][1] = off + b;
            pl.block_bytes[mu] = b;
            off += 2 * b;
        }
        pl.total_bytes = off;
        DevBuf send;
        CUDA_TRY(cudaMalloc(&send.p, (size_t)off), "cudaMalloc(link halo send)");
        CUDA_TRY(cudaMalloc(&l->aux, (size_t)off), "cudaMalloc(link halo)");
        CUDA_TRY(cudaMemsetAsync(send.p, 0, (size_t)off, s), "cudaMemsetAsync");
        CUDA_TRY(launch_lhalo_pack(full->prec, c->nvec, l->base, send.p, c->kg, l->lhoff, s), "link halo pack");
        std::string err;
        r = halo_exchange_buf(c, pl, send.p, l->aux, s, err);
        if (r != CD_OK) return fail(r, err);
        CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
    if (max_dev) {
        DevBuf d;
        CUDA_TRY(cudaMalloc(&d.p, sizeof(float)), "cudaMalloc");
        float *dv = static_cast<float *>(d.p);
        CUDA_TRY(cudaMemsetAsync(dv, 0, sizeof(float), s), "cudaMemsetAsync");
        CUDA_TRY(launch_hermdev(full->prec, c->nvec, full->base, c->kg, dv, s, l->aux, l->aux ? l->lhoff : nullptr),
                 "hermiticity check");
        float h = 0.0f;
        CUDA_TRY(cudaMemcpyAsync(&h, dv, sizeof(float), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
        CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        *max_dev = h;
    }
    *out = guard.release();
    return CD_OK;
    API_END
}

int coarse_links_upload(cd_context *c, cd_precision p, const void *src, int src_on_device, cd_host_dtype dt,
                        void *stream, cd_links **out)
{
    API_BEGIN
    if (!c || !src || !out) return fail(CD_ERR_INVALID, "ctx/src/out is NULL");
    CTX_GUARD(c);
    if (p != CD_FP32 && p != CD_FP16) return fail(CD_ERR_INVALID, "bad precision");
    if (dt != CD_C64 && dt != CD_C128) return fail(CD_ERR_INVALID, "bad dtype");
    cd_links *l = nullptr;
    int r = links_new(c, p, &l);
    if (r != CD_OK) return r;
    cudaStream_t s = S(stream);
    const size_t elem = dt == CD_C128 ? 16 : 8;
    const size_t mat_src = elem * c->N * c->N;
    const int64_t nmats = 9 * c->V;
    if (src_on_device) {
        cudaError_t e = launch_links_convert(p, c->nvec, nmats, src, dt == CD_C128, l->base, s, 0);
        if (e != cudaSuccess) {
            cudaFree(l->base);
            delete l;
            return cuda_fail(e, "links convert");
        }
    } else {
        // stage through a bounded device buffer (<= 64 MB of source per chunk)
        const int64_t chunk = std::max<int64_t>(1, (int64_t)((64u << 20) / mat_src));
        void *stage = nullptr;
        cudaError_t e = cudaMalloc(&stage, (size_t)std::min<int64_t>(chunk, nmats) * mat_src);
        if (e != cudaSuccess) {
            cudaFree(l->base);
            delete l;
            return fail(CD_ERR_OOM, "cudaMalloc(stage)");
        }
        for (int64_t m0 = 0; m0 < nmats && e == cudaSuccess; m0 += chunk) {
            const int64_t n = std::min(chunk, nmats - m0);
            e = cudaMemcpyAsync(stage, static_cast<const unsigned char *>(src) + m0 * mat_src, n * mat_src,
                                cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = launch_links_convert(p, c->nvec, n, stage, dt == CD_C128, l->base, s, m0);
        }
        cudaError_t e2 = cudaStreamSynchronize(s);
        cudaFree(stage);
        if (e == cudaSuccess) e = e2;
        if (e != cudaSuccess) {
            cudaFree(l->base);
            delete l;
            return cuda_fail(e, "links upload");
        }
    }
    *out = l;
    return CD_OK;
    API_END
}

int coarse_links_generate(cd_context *c, cd_precision p, int kind, uint64_t seed, int32_t scale_log2, void *stream,
                          cd_links **out)
{
    API_BEGIN
    if (!c || !out) return fail(CD_ERR_INVALID, "ctx/out is NULL");
    CTX_GUARD(c);
    if (p != CD_FP32 && p != CD_FP16) return fail(CD_ERR_INVALID, "bad precision");
    if (kind < 0 || kind > 3) return fail(CD_ERR_INVALID, "bad links kind");
    if (scale_log2 < -60 || scale_log2 > 60) return fail(CD_ERR_INVALID, "scale_log2 out of range");
    cd_links *l = nullptr;
    int r = links_new(c, p, &l);
    if (r != CD_OK) return r;
    cudaError_t e = launch_links_generate(p, c->nvec, c, kind, seed, scale_log2, l->base, S(stream));
    if (e != cudaSuccess) {
        cudaFree(l->base);
        delete l;
        return cuda_fail(e, "links generate");
    }
    *out = l;
    return CD_OK;
    API_END
}

size_t coarse_links_stored_bytes(const cd_links *l)
{
    if (!l || l->eo) return 0;
    const size_t nm = (l->compressed ? 5 : 9) * (size_t)l->ctx->V;
    const size_t NN = (size_t)l->ctx->N * l->ctx->N;
    return l->prec == CD_FP32 ? 8 * NN * nm : 4 * NN * nm + 4 * nm;
}

int coarse_links_read_stored(const cd_links *l, void *dst, int dst_on_device, void *stream)
{
    API_BEGIN
    if (!l || !dst) return fail(CD_ERR_INVALID, "links/dst is NULL");
    if (l->eo) return fail(CD_ERR_INVALID, "even-odd prepared links have no canonical stored form");
    CTX_GUARD(l->ctx);
    const size_t NN = (size_t)l->ctx->N * l->ctx->N;
    const bool f16 = l->prec == CD_FP16;
    return read_stored(l->base, (l->compressed ? 5 : 9) * l->ctx->V, f16 ? 4 * NN : 8 * NN,
                       mat_rec_bytes(l->ctx->N, l->prec), f16, dst, dst_on_device, S(stream));
    API_END
}

int coarse_links_free(cd_links *l)
{
    API_BEGIN
    if (!l) return fail(CD_ERR_INVALID, "links is NULL");
    if (l->aux) cudaFree(l->aux);
    if (l->tbuf) cudaFree(l->tbuf);
    cudaFree(l->base);
    delete l;
    return CD_OK;
    API_END
}

// ------------------------------------------------------------------ apply
static int check_objs(const cd_links *l, const cd_field *out, const cd_field *in)
{
    if (!l || !out || !in) return fail(CD_ERR_INVALID, "links/out/in is NULL");
    if (l->ctx != out->ctx || l->ctx != in->ctx) return fail(CD_ERR_MISMATCH, "objects from different contexts");
    if (l->prec != out->prec || l->prec != in->prec) return fail(CD_ERR_MISMATCH, "precision mismatch");
    if (out->base == in->base) return fail(CD_ERR_INVALID, "out must not alias in");
    if (out->nrhs != 1 || in->nrhs != 1) return fail(CD_ERR_INVALID, "multi-RHS fields need coarse_dslash_apply_mrhs");
    if (out->parity >= 0 || in->parity >= 0) return fail(CD_ERR_INVALID, "parity fields need coarse_dslash_apply_eo");
    if (l->eo) return fail(CD_ERR_INVALID, "even-odd prepared links need coarse_dslash_apply_eo");
    const char *ob = static_cast<const char *>(out->base), *ib = static_cast<const char *>(in->base);
    const size_t need = coarse_field_bytes(l->ctx, l->prec);
    if (ob < ib + need && ib < ob + need) return fail(CD_ERR_INVALID, "out overlaps in");
    return CD_OK;
}

// Pick the kernel variant for (prec, dagger): forced > cached > tuned > heuristic.
// Tuning (first call of a key, "auto-tuned upon first call and cached") times
// every variant with CUDA events on the caller's stream; trial launches write `out` only.
// Every dslash launch gets the next sequence number (the ring kernel's ticket slot).
// While an NCCL halo exchange is in flight the persistent interior kernel leaves
// CD_OPT_NCCL_SM_RESERVE SMs free: NCCL's copy kernels need SMs to make progress, and the ring
// (one 227 KB CTA per SM) would otherwise hold every SM until the interior is done.
static cudaError_t launch_next(cd_context *c, cd_precision p, int id, ApplyArgs a, cudaStream_t s, bool pdl)
{
    a.seq = c->seq++;
    int sms = (a.halo && transport_of(c) == TR_NCCL) ? c->num_sms - c->nccl_sm_reserve : c->num_sms;
    static const int cap = getenv("CD_RING_SMS") ? atoi(getenv("CD_RING_SMS")) : 0;   // diagnostic: persistent grid cap
    if (cap > 0 && cap < sms) sms = cap;
    return launch_dslash(p, id, a, s, pdl, sms);
}

// Split (multi-rank or self-halo) apply: pack (+ transfer) on the high-priority
// comm stream overlapped with the interior kernel on s, then -- once the halo has landed -- the
// halo-term kernel for the remote hops of the face sites.
extern "C++" {
template <class Interior, class Term>
static int run_split(cd_context *c, cd_precision p, const void *in, ApplyArgs &a, cudaStream_t s, Interior interior,
                     Term term)
{
    const cd_halo_plan pl = ctx_plan(c, p);
    std::string err;
    if (transport_of(c) == TR_PEER) {   // exchange epochs are host counters baked into the launches
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        if (cap != cudaStreamCaptureStatusNone)
            return fail(CD_ERR_UNSUPPORTED, "peer-transport applies cannot be captured in a CUDA graph (per-exchange epochs)");
    }
    HaloX x;
    int r = halo_begin(c, pl, &x, err);
    if (r != CD_OK) return fail(r, err);
    a.recv = x.recv;
    CUDA_TRY(cudaEventRecord(c->ev_in, s), "cudaEventRecord");
    CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_in, 0), "cudaStreamWaitEvent");
    CUDA_TRY(launch_pack(p, c->nvec, in, x.pd, a.g, c->comm_stream), "halo pack");
    r = halo_post(c, pl, x, c->comm_stream, err);
    if (r != CD_OK) return fail(r, err);
    CUDA_TRY(cudaEventRecord(c->ev_halo, c->comm_stream), "cudaEventRecord");
    CUDA_TRY(interior(), "dslash interior launch");
    CUDA_TRY(cudaStreamWaitEvent(s, c->ev_halo, 0), "cudaStreamWaitEvent");
    r = halo_finish(c, x, s, err);
    if (r != CD_OK) return fail(r, err);
    CUDA_TRY(term(), "halo kernel");
    return CD_OK;
}
}  // extern "C++"

static int resolve_variant(cd_context *c, cd_precision p, int dag, const ApplyArgs &a, cudaStream_t s, int *id)
{
    const int nvar = variant_count(p, c->nvec);
    if (c->force_variant >= 0) {
        if (c->force_variant >= nvar) return fail(CD_ERR_INVALID, "forced variant out of range for this precision");
        *id = c->force_variant;
        return CD_OK;
    }
    TuneKey key{(int)p, dag};
    {
        std::lock_guard<std::mutex> lk(c->mu);
        auto it = c->chosen.find(key);
        if (it != c->chosen.end()) {
            *id = it->second;
            return CD_OK;
        }
    }
    const std::string ks = tune_key_str(c, (int)p, dag);
    int v = tune_file_lookup(ks);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    if (v < 0 || v >= nvar) {
        v = variant_heuristic(p, c->nvec, a.g, c->num_sms);
        if (c->tune && cap == cudaStreamCaptureStatusNone) {
            cudaEvent_t e0, e1;
            CUDA_TRY(cudaEventCreate(&e0), "event");
            CUDA_TRY(cudaEventCreate(&e1), "event");
            float best = 1e30f;
            const int reps = c->V >= 2048 ? 3 : 20;
            // time `r` back-to-back launches of variant id2 with the production PDL setting (a
            // variant that overlaps its ramp with the previous launch's tail is timed as it will
            // run in a chain of applies); < 0 if it cannot run here
            const bool tpdl = c->pdl != 0;
            // L2-resident lattices (the latency regime): eager back-to-back launches would time the
            // host's launch rate, so r applies are captured in a CUDA graph on a private stream
            // (PDL edges kept) and the graph's replay is timed -- how a solver runs them
            const double lbytes = (double)c->V * 9.0 * (p == CD_FP32 ? 8.0 : 4.0) * c->N * c->N;
            const bool graph_tune = lbytes <= 64e6 && !getenv("CD_TUNE_EAGER");
            cudaStream_t ts = nullptr;
            cudaEvent_t evs = nullptr;
            if (graph_tune) {
                if (cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&evs, cudaEventDisableTiming) != cudaSuccess)
                    return fail(CD_ERR_CUDA, "tuner stream");
                cudaEventRecord(evs, s);
                cudaStreamWaitEvent(ts, evs, 0);   // trials after the caller's prior work
            }
            auto timeit_graph = [&](int id2, int r) -> float {
                cudaGraph_t gr = nullptr;
                cudaGraphExec_t ge = nullptr;
                if (cudaStreamBeginCapture(ts, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                    cudaGetLastError();
                    return -1.f;
                }
                cudaError_t e = cudaSuccess;
                for (int rr = 0; rr < r && e == cudaSuccess; rr++) e = launch_next(c, p, id2, a, ts, tpdl);
                cudaError_t e2 = cudaStreamEndCapture(ts, &gr);
                if (e == cudaSuccess) e = e2;
                if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, gr, 0);
                float ms = -1.f;
                if (e == cudaSuccess) e = cudaGraphLaunch(ge, ts);   // warm-up
                if (e == cudaSuccess) e = cudaEventRecord(e0, ts);
                if (e == cudaSuccess) e = cudaGraphLaunch(ge, ts);
                if (e == cudaSuccess) e = cudaEventRecord(e1, ts);
                if (e == cudaSuccess) e = cudaEventSynchronize(e1);
                if (e == cudaSuccess) {
                    cudaEventElapsedTime(&ms, e0, e1);
                    ms /= r;
                } else {
                    cudaGetLastError();
                    ms = -1.f;
                }
                if (ge) cudaGraphExecDestroy(ge);
                if (gr) cudaGraphDestroy(gr);
                return ms;
            };
            auto timeit = [&](int id2, int r) -> float {
                if (graph_tune) return timeit_graph(id2, std::max(r, 50));
                cudaError_t e = cudaSuccess;
                for (int w = 0; w < 2 && e == cudaSuccess; w++) e = launch_next(c, p, id2, a, s, tpdl);
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    return -1.f;
                }
                cudaEventRecord(e0, s);
                for (int rr = 0; rr < r && e == cudaSuccess; rr++) e = launch_next(c, p, id2, a, s, tpdl);
                cudaEventRecord(e1, s);
                if (e != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess) {
                    cudaGetLastError();
                    return -1.f;
                }
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                return ms / r;
            };
            // pass 1: every variant briefly; pass 2: the three fastest re-timed in interleaved
            // rounds (min over rounds), so clock ramps and run-to-run noise do not pick the winner
            std::vector<std::pair<float, int>> t1;
            for (int id2 = 0; id2 < nvar; id2++) {
                const float ms = timeit(id2, reps);
                if (ms >= 0.f) t1.emplace_back(ms, id2);
            }
            std::sort(t1.begin(), t1.end());
            if (t1.size() > 3) t1.resize(3);
            std::vector<float> t2(t1.size(), 1e30f);
            const double link_bytes = (double)c->V * 9.0 * (p == CD_FP32 ? 8.0 : 4.0) * c->N * c->N;
            const bool hbm = link_bytes > 128e6;   // links stream from HBM (larger than L2)
            if (hbm && !t1.empty()) {
                // HBM-streaming sizes run power-capped in any sustained use (a solver, the bench),
                // and the variants rank differently there than in a short full-clock burst
                // (profiles/r02/sustained_variants.jsonl): heat the GPU for ~0.3 s, then compare the
                // finalists in interleaved ~60 ms windows and keep the median of five rounds
                const float ms1 = std::max(t1[0].first, 1e-3f);
                timeit(t1[0].second, std::max(4, (int)(300.f / ms1)));
                const int r2 = std::max(2 * reps + 4, (int)(60.f / ms1));
                std::vector<std::vector<float>> rr(t1.size());
                for (int round = 0; round < 5; round++)
                    for (size_t i = 0; i < t1.size(); i++) {
                        const float ms = timeit(t1[i].second, r2);
                        if (ms >= 0.f) rr[i].push_back(ms);
                    }
                for (size_t i = 0; i < t1.size(); i++)
                    if (!rr[i].empty()) {
                        std::sort(rr[i].begin(), rr[i].end());
                        t2[i] = rr[i][rr[i].size() / 2];
                    }
            } else {
                for (int round = 0; round < 3; round++)
                    for (size_t i = 0; i < t1.size(); i++) {
                        const float ms = timeit(t1[i].second, 2 * reps + 4);
                        if (ms >= 0.f) t2[i] = std::min(t2[i], ms);
                    }
            }
            for (size_t i = 0; i < t1.size(); i++)
                if (t2[i] < best) best = t2[i], v = t1[i].second;
            // Near-ties on lattices whose links stream from HBM go to the TMA ring: it moves the links
            // without a register round trip and
            // draws less power per byte, so under the sustained power cap of a long run it keeps
            // a higher SM clock (8^4 fp32, 2000 steps: 96.2 vs 98.2 us per apply for fg_kw3_wr4,
            // profiles/r01/bench_sustained_variants.txt) -- a difference the short tuning bursts
            // at full clock cannot see.
            // a split context on the peer transport runs a ring as ONE fused launch, any other variant
            // as pack + interior + wait + halo-term kernels the trials above do not include (the
            // trials time the interior only -- an exchange needs every rank): measured on M5's T
            // split that costs the unfused path ~8-10 %, so rings win within 8 %
            const float tie = (a.halo && transport_of(c) == TR_PEER && c->fuse_split) ? 1.08f : 1.015f;
            if ((hbm || tie > 1.05f) && std::strncmp(variant_name(p, c->nvec, v), "ring", 4) != 0)
                for (size_t i = 0; i < t1.size(); i++)
                    if (std::strncmp(variant_name(p, c->nvec, t1[i].second), "ring", 4) == 0 && t2[i] <= tie * best) {
                        v = t1[i].second;
                        best = t2[i];
                        break;
                    }
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            if (ts) {
                cudaStreamSynchronize(ts);
                cudaStreamDestroy(ts);
            }
            if (evs) cudaEventDestroy(evs);
            tune_file_store(ks, v, variant_name(p, c->nvec, v), best * 1000.f);
        }
    }
    {
        std::lock_guard<std::mutex> lk(c->mu);
        c->chosen[key] = v;
    }
    *id = v;
    return CD_OK;
}

static int do_apply(const cd_links *l, cd_field *out, const cd_field *in, void *stream, int dag)
{
    int r = check_objs(l, out, in);
    if (r != CD_OK) return r;
    cd_context *c = l->ctx;
    CTX_GUARD(c);
    cudaStream_t s = S(stream);
    if (l->compressed && l->split != c->kg.split)
        return fail(CD_ERR_INVALID, "compressed links were built under a different halo split (set CD_OPT_HALO_SELF_MASK "
                                    "before coarse_links_compress_hermitian)");
    c->applied = true;
    {
        std::string err;
        r = transport_check(c, err);
        if (r != CD_OK) return fail(r, err);
    }
    ApplyArgs a{};
    a.links = l->base;
    a.in = in->base;
    a.out = out->base;
    a.nvec = c->nvec;
    a.dagger = dag;
    const bool halo = c->kg.split != 0;
    if (l->compressed) {   // tau3-hermitian compressed links (NEXT-2)
        a.ysplit = c->ysplit;       // fp16: whole-site re-quantisation scratch
        a.site_cnt = c->site_cnt;
        if (!halo) {
            a.g = c->kg;
            // fp16 on large lattices: the persistent TMA ring reading backward links transposed (HBM
            // carries 5 matrices per site): 1.7x the fine-grained fgh16 kernel and 3-5 % faster than
            // the full 9-matrix apply; fp32 (and small lattices): the fine-grained fgh kernel, which
            // beats the ring there (81.6 vs 103.6 us at 8^4, profiles/r02/compressed_ring.txt)
            static const int comp_ring = getenv("CD_COMP_RING") ? atoi(getenv("CD_COMP_RING")) : -1;
            // fp16 only: the fp32 compressed ring (CD_COMP_RING=1 used to force it) shows intermittent
            // errors of 1e-4..1e-2 on repeated applies (also in the round-2 build before the stage
            // reorder; the fp16 ring is bit-stable), so fp32 always takes the fine-grained kernel
            const bool use_ring = l->prec == CD_FP16 && comp_ring != 0;
            if (use_ring && c->V >= 4 * c->num_sms) {
                a.work = c->work;
                a.seq = c->seq++;
                static const int mps_env = getenv("CD_COMP_MPS") ? atoi(getenv("CD_COMP_MPS")) : 3;
                // two CTAs per SM for the three-matrix compressed ring (its consumers' transposed column
                // reads are latency bound: twice the consumer warps per SM): M5 fp16 1617 -> 1456 us, 8^4
                // 49.8 -> 45.7 us (profiles/r02/compressed_2cta_ab.txt); CD_COMP_2CTA=0: one CTA per SM
                const int two = getenv("CD_COMP_2CTA") ? atoi(getenv("CD_COMP_2CTA")) : 1;
                const int mps = (mps_env == 9 && l->prec == CD_FP16 && c->nvec == 24) ? 9 : (two == 1 ? 103 : 3);
                CUDA_TRY(launch_ringh(l->prec, a, s, c->pdl != 0, c->num_sms, mps), "compressed ring launch");
                return CD_OK;
            }
            CUDA_TRY(launch_fgh(l->prec, a, s, c->pdl != 0), "compressed dslash launch");
            return CD_OK;
        }
        // multi-rank: vector halo as for the full operator; remote backward hops use the link halo
        a.g = halo_geom(c, l->prec);
        a.halo = 1;
        a.scratch = c->face_scratch;
        a.face_sites = c->face_sites;
        a.n_face = c->n_face;
        a.lhalo = l->aux;
        for (int mu = 0; mu < 4; mu++) a.lhoff[mu] = l->lhoff[mu];
        return run_split(
            c, l->prec, in->base, a, s, [&] { return launch_fgh(l->prec, a, s, false); },
            [&] { return launch_fgh_halo(l->prec, a, s); });
    }
    a.g = halo ? halo_geom(c, l->prec) : c->kg;
    a.halo = halo ? 1 : 0;
    a.scratch = c->face_scratch;
    a.recv = c->recv_buf;
    a.face_sites = c->face_sites;
    a.n_face = c->n_face;
    a.work = c->work;
    a.ysplit = c->ysplit;
    a.site_cnt = c->site_cnt;
    a.chain_cnt = c->chain_cnt;
    int id = 0;
    r = resolve_variant(c, l->prec, dag, a, s, &id);
    if (r != CD_OK) return r;
    if (!halo) {
        CUDA_TRY(launch_next(c, l->prec, id, a, s, c->pdl != 0), "dslash launch");
        return CD_OK;
    }
    int kw = 0, wr = 0;
    if (transport_of(c) == TR_PEER && variant_kind(l->prec, c->nvec, id, &kw, &wr) == 0 && c->fuse_split) {
        // fused split apply: ONE persistent launch packs its face slices straight
        // into the neighbours' windows, streams the interior sites, then the face sites with
        // their remote records read from this rank's window after an in-kernel arrival wait
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        if (cap != cudaStreamCaptureStatusNone)
            return fail(CD_ERR_UNSUPPORTED, "peer-transport applies cannot be captured in a CUDA graph (per-exchange epochs)");
        const cd_halo_plan pl = ctx_plan(c, l->prec);
        std::string err;
        HaloX x;
        r = halo_begin(c, pl, &x, err);
        if (r != CD_OK) return fail(r, err);
        a.fused = 1;
        a.pd = x.pd;
        a.recv = x.recv;
        a.wflag = reinterpret_cast<const unsigned long long *>(c->win);
        a.wmask = x.mask;
        a.wtarget = x.target;
        a.wtimeout = c->peer_timeout_ns;
        a.werr = c->err_dev;
        a.pack_cnt = c->pack_cnt;
        a.rot = (c->kg.split == 8) ? (int)(c->V / c->local[3]) : 0;
        CUDA_TRY(launch_next(c, l->prec, id, a, s, c->pdl != 0), "fused split apply");
        return CD_OK;
    }
    return run_split(
        c, l->prec, in->base, a, s, [&] { return launch_next(c, l->prec, id, a, s, false); },
        [&] { return launch_halo(l->prec, a, s); });
}

int coarse_dslash_apply(const cd_links *l, cd_field *out, const cd_field *in, void *stream)
{
    API_BEGIN
    return do_apply(l, out, in, stream, 0);
    API_END
}

int coarse_dslash_apply_dagger(const cd_links *l, cd_field *out, const cd_field *in, void *stream)
{
    API_BEGIN
    return do_apply(l, out, in, stream, 1);
    API_END
}

// ------------------------------------------------------------------ even-odd (NEXT-3)
// Even local extents: local parity == global parity (the rank origins are even) and every x0
// pair holds one site of each parity.
static bool eo_geometry_ok(const cd_context *c)
{
    for (int mu = 0; mu < 4; mu++)
        if (c->local[mu] % 2) return false;
    return true;
}

// The even-odd stages reuse the full operator's fp32 vector-halo plan and transport.
struct EoExchange {
    cd_context *c;
    cd_halo_plan pl;
    HaloX x;
    cudaStream_t s;
    int status = CD_OK;
    std::string err;
};
static cudaError_t eo_begin(void *p, PackDst *pd, const void **recv)
{
    EoExchange *e = static_cast<EoExchange *>(p);
    e->status = halo_begin(e->c, e->pl, &e->x, e->err);
    *pd = e->x.pd;
    *recv = e->x.recv;
    return e->status == CD_OK ? cudaSuccess : cudaErrorUnknown;
}
static cudaError_t eo_post(void *p)
{
    EoExchange *e = static_cast<EoExchange *>(p);
    e->status = halo_post(e->c, e->pl, e->x, e->c->comm_stream, e->err);
    return e->status == CD_OK ? cudaSuccess : cudaErrorUnknown;
}
static cudaError_t eo_finish(void *p)
{
    EoExchange *e = static_cast<EoExchange *>(p);
    e->status = halo_finish(e->c, e->x, e->s, e->err);
    return e->status == CD_OK ? cudaSuccess : cudaErrorUnknown;
}

size_t coarse_field_bytes_parity(const cd_context *c, cd_precision p)
{
    if (!c || (p != CD_FP32 && p != CD_FP16)) return 0;
    return align256(vec_rec_bytes(c->N, p) * (size_t)(c->V / 2));
}

int coarse_field_alloc_parity(cd_context *c, cd_precision p, int parity, void *mem, size_t bytes, cd_field **out)
{
    API_BEGIN
    if (!c || !out) return fail(CD_ERR_INVALID, "ctx/out is NULL");
    if (p != CD_FP32 && p != CD_FP16) return fail(CD_ERR_INVALID, "bad precision");
    if (parity != 0 && parity != 1) return fail(CD_ERR_INVALID, "parity must be 0 (even) or 1 (odd)");
    CTX_GUARD(c);
    if (!eo_geometry_ok(c)) return fail(CD_ERR_UNSUPPORTED, "even-odd needs every local L_mu even");
    const size_t need = coarse_field_bytes_parity(c, p);
    bool owned = false;
    if (!mem) {
        CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
        cudaError_t e = cudaMalloc(&mem, need);
        if (e != cudaSuccess) return fail(CD_ERR_OOM, std::string("cudaMalloc(field): ") + cudaGetErrorString(e));
        bytes = need;
        owned = true;
    } else {
        if (reinterpret_cast<uintptr_t>(mem) % 256) return fail(CD_ERR_INVALID, "device_mem must be 256-B aligned");
        if (bytes < need) return fail(CD_ERR_INVALID, "device_mem too small (need coarse_field_bytes_parity)");
    }
    *out = new cd_field{c, p, mem, bytes, owned, 1, parity};
    return CD_OK;
    API_END
}

int coarse_links_prepare_eo(const cd_links *full, void *stream, cd_links **out)
{
    API_BEGIN
    if (!full || !out) return fail(CD_ERR_INVALID, "links/out is NULL");
    CTX_GUARD(full->ctx);
    if (full->compressed || full->eo) return fail(CD_ERR_INVALID, "needs full (uncompressed) links");
    if (full->prec != CD_FP32) return fail(CD_ERR_UNSUPPORTED, "even-odd: fp32 storage only");
    cd_context *c = full->ctx;
    if (!eo_geometry_ok(c)) return fail(CD_ERR_UNSUPPORTED, "even-odd needs every local L_mu even");
    cudaStream_t s = S(stream);
    const size_t mrec = mat_rec_bytes(c->N, CD_FP32);
    const size_t half = (size_t)(c->V / 2);
    DevBuf even, odd, t, sing;
    CUDA_TRY(cudaMalloc(&even.p, align256(half * 9 * mrec)), "cudaMalloc(eo even)");
    CUDA_TRY(cudaMalloc(&odd.p, align256(half * 8 * mrec)), "cudaMalloc(eo odd)");
    CUDA_TRY(cudaMalloc(&t.p, align256(half * vec_rec_bytes(c->N, CD_FP32))), "cudaMalloc(eo t)");
    CUDA_TRY(cudaMalloc(&sing.p, sizeof(int)), "cudaMalloc");
    int *sg = static_cast<int *>(sing.p);
    CUDA_TRY(cudaMemsetAsync(sg, 0, sizeof(int), s), "cudaMemsetAsync");
    CUDA_TRY(launch_eo_prepare(c->nvec, full->base, even.p, odd.p, c->kg, sg, s), "eo prepare");
    int hs = 0;
    CUDA_TRY(cudaMemcpyAsync(&hs, sg, sizeof(int), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    if (hs) return fail(CD_ERR_INVALID, "a diagonal block X on an odd site is singular");
    void *ev = even.release(), *od = odd.release(), *tb = t.release();
    *out = new cd_links{c, CD_FP32, ev, align256(half * 9 * mrec), 0, 1, od, tb};
    return CD_OK;
    API_END
}

int coarse_dslash_apply_eo(const cd_links *l, cd_field *out, const cd_field *in, int dagger, void *stream)
{
    API_BEGIN
    if (!l || !out || !in) return fail(CD_ERR_INVALID, "links/out/in is NULL");
    CTX_GUARD(l->ctx);
    if (!l->eo) return fail(CD_ERR_INVALID, "links not prepared with coarse_links_prepare_eo");
    if (l->ctx != out->ctx || l->ctx != in->ctx) return fail(CD_ERR_MISMATCH, "objects from different contexts");
    if (out->parity != 0 || in->parity != 0) return fail(CD_ERR_INVALID, "in/out must be even-parity fields");
    if (out->prec != CD_FP32 || in->prec != CD_FP32) return fail(CD_ERR_MISMATCH, "even-odd: fp32 fields");
    if (out->base == in->base) return fail(CD_ERR_INVALID, "out must not alias in");
    cd_context *c = l->ctx;
    c->applied = true;
    {
        std::string err;
        const int r = transport_check(c, err);
        if (r != CD_OK) return fail(r, err);
    }
    EoApply e{};
    e.even = l->base;
    e.odd = l->aux;
    e.in_e = in->base;
    e.t_o = l->tbuf;
    e.out_e = out->base;
    e.dagger = dagger ? 1 : 0;
    e.s = S(stream);
    e.pdl = c->pdl != 0;
    e.halo = c->kg.split != 0 ? 1 : 0;
    e.g = e.halo ? halo_geom(c, CD_FP32) : c->kg;
    EoExchange ex{c, ctx_plan(c, CD_FP32), {}, e.s};
    if (e.halo) {
        e.comm_stream = c->comm_stream;
        e.ev_in = c->ev_in;
        e.ev_halo = c->ev_halo;
        e.scratch = c->face_scratch;
        e.face_sites = c->face_sites;
        e.n_face = c->n_face;
        e.begin = eo_begin;
        e.post = eo_post;
        e.finish = eo_finish;
        e.exchange_arg = &ex;
    }
    const cudaError_t ce = launch_eo_apply(c->nvec, e);
    if (ex.status != CD_OK) return fail(ex.status, ex.err);
    CUDA_TRY(ce, "eo apply");
    return CD_OK;
    API_END
}

int coarse_dslash_apply_mrhs(const cd_links *l, cd_field *out, const cd_field *in, int dagger, void *stream)
{
    API_BEGIN
    if (!l || !out || !in) return fail(CD_ERR_INVALID, "links/out/in is NULL");
    CTX_GUARD(l->ctx);
    if (l->ctx != out->ctx || l->ctx != in->ctx) return fail(CD_ERR_MISMATCH, "objects from different contexts");
    if (l->compressed || l->eo) return fail(CD_ERR_INVALID, "apply_mrhs needs full (uncompressed, not even-odd) links");
    if (out->parity >= 0 || in->parity >= 0) return fail(CD_ERR_INVALID, "apply_mrhs needs full-lattice fields");
    if (l->prec != CD_FP16 || out->prec != CD_FP16 || in->prec != CD_FP16)
        return fail(CD_ERR_UNSUPPORTED, "the tensor-core multi-RHS path needs fp16 storage (links and fields)");
    if (in->nrhs != out->nrhs) return fail(CD_ERR_MISMATCH, "nrhs mismatch");
    if (in->nrhs % 128) return fail(CD_ERR_UNSUPPORTED, "nrhs must be a multiple of 128");
    if (out->base == in->base) return fail(CD_ERR_INVALID, "out must not alias in");
    cd_context *c = l->ctx;
    c->applied = true;
    cudaStream_t s = S(stream);
    if (c->kg.split == 0) {
        CUDA_TRY(launch_mrhs(c->nvec, l->base, in->base, out->base, c->kg, in->nrhs, dagger ? 1 : 0, s, c->num_sms),
                 "mrhs launch");
        return CD_OK;
    }
    // multi-rank: the face blocks of every split dim travel in the tensor-core layout
    // ([f][rhs block] records of 128 rhs); the interior sites run while the exchange is in flight,
    // the face sites after it (their remote hops read the receive buffer).
    {
        std::string err;
        const int r = transport_check(c, err);
        if (r != CD_OK) return fail(r, err);
    }
    const int nrb = in->nrhs / 128;
    const size_t blk = (size_t)128 * 4 * c->N + 16;
    cd_halo_plan pl = ctx_plan(c, CD_FP16);
    MrhsHalo hl{};
    int64_t off = 0;
    for (int mu = 0; mu < 4; mu++) {
        pl.block_offset[mu][0] = pl.block_offset[mu][1] = 0;
        pl.block_bytes[mu] = 0;
        if (!((c->kg.split >> mu) & 1)) continue;
        const int64_t b = (int64_t)(c->V / c->local[mu]) * nrb * (int64_t)blk;
        pl.block_offset[mu][0] = hl.off[mu][0] = off;
        pl.block_offset[mu][1] = hl.off[mu][1] = off + b;
        pl.block_bytes[mu] = b;
        off += 2 * b;
    }
    pl.total_bytes = off;
    if ((size_t)off > c->mrhs_cap) {
        if (c->mrhs_send) cudaFree(c->mrhs_send);
        if (c->mrhs_recv) cudaFree(c->mrhs_recv);
        c->mrhs_send = c->mrhs_recv = nullptr;
        c->mrhs_cap = 0;
        CUDA_TRY(cudaMalloc(&c->mrhs_send, (size_t)off), "cudaMalloc(mrhs send)");
        CUDA_TRY(cudaMalloc(&c->mrhs_recv, (size_t)off), "cudaMalloc(mrhs recv)");
        c->mrhs_cap = (size_t)off;
    }
    hl.recv = c->mrhs_recv;
    CUDA_TRY(cudaEventRecord(c->ev_in, s), "cudaEventRecord");
    CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_in, 0), "cudaStreamWaitEvent");
    CUDA_TRY(launch_mrhs_pack(c->nvec, in->base, c->mrhs_send, c->kg, in->nrhs, hl, c->comm_stream), "mrhs pack");
    {
        std::string err;
        const int r = halo_exchange_buf(c, pl, c->mrhs_send, c->mrhs_recv, c->comm_stream, err);
        if (r != CD_OK) return fail(r, err);
    }
    CUDA_TRY(cudaEventRecord(c->ev_halo, c->comm_stream), "cudaEventRecord");
    CUDA_TRY(launch_mrhs(c->nvec, l->base, in->base, out->base, c->kg, in->nrhs, dagger ? 1 : 0, s, c->num_sms,
                         c->interior_sites, c->n_interior, &hl),
             "mrhs interior launch");
    CUDA_TRY(cudaStreamWaitEvent(s, c->ev_halo, 0), "cudaStreamWaitEvent");
    CUDA_TRY(launch_mrhs(c->nvec, l->base, in->base, out->base, c->kg, in->nrhs, dagger ? 1 : 0, s, c->num_sms,
                         c->face_sites, c->n_face, &hl),
             "mrhs face launch");
    return CD_OK;
    API_END
}

// One chain launch of variant `id`; advances the context's counter base on success.
static cudaError_t chain_launch(cd_context *c, cd_precision p, int id, const ApplyArgs &a, int n, cudaStream_t s)
{
    int nrb = 0;
    const bool ll = id >= LL_CHAIN_ID0;
    cudaError_t e = launch_chain(p, id, a, n, ll ? c->ll_base : c->chain_base, s, c->num_sms, &nrb);
    if (e == cudaSuccess) {
        if (ll) c->ll_base += (unsigned)n;   // epochs ll_base+1 .. ll_base+n used
        else c->chain_base += (unsigned)(n * nrb);
    }
    return e;
}

int coarse_dslash_apply_chain(const cd_links *l, cd_field *x, cd_field *y, int n, int dagger, void *stream)
{
    API_BEGIN
    int r = check_objs(l, y, x);
    if (r != CD_OK) return r;
    if (l->compressed) return fail(CD_ERR_INVALID, "apply_chain needs full (uncompressed) links");
    if (n < 0) return fail(CD_ERR_INVALID, "n must be >= 0");
    cd_context *c = l->ctx;
    CTX_GUARD(c);
    if (c->kg.split != 0) return fail(CD_ERR_UNSUPPORTED, "apply_chain is single-rank (no halo split)");
    if (n == 0) return CD_OK;
    cudaStream_t s = S(stream);
    c->applied = true;
    ApplyArgs a{};
    a.links = l->base;
    a.in = x->base;
    a.out = y->base;
    a.nvec = c->nvec;
    a.dagger = dagger ? 1 : 0;
    a.g = c->kg;
    a.chain_cnt = c->chain_cnt;
    if (!c->llbuf) {   // 2 x V LL records of at most 16N bytes, zeroed (epoch 0 is never awaited)
        const size_t llb = 2 * (size_t)c->V * 16 * c->N;
        CUDA_TRY(cudaMalloc(&c->llbuf, llb), "cudaMalloc(llbuf)");
        CUDA_TRY(cudaMemset(c->llbuf, 0, llb), "cudaMemset(llbuf)");
    }
    a.llbuf = c->llbuf;
    a.poll_ns = 0;
    if (const char *ev = getenv("CD_POLL_NS")) a.poll_ns = atoi(ev);
    a.poll_d0 = 300;   // measured best at 2^4 (profiles/r01/chain_llreg.jsonl)
    a.poll_d1 = 0;
    if (const char *ev = getenv("CD_POLL_D0")) a.poll_d0 = atoi(ev);
    if (const char *ev = getenv("CD_POLL_D1")) a.poll_d1 = atoi(ev);
    const cd_precision p = l->prec;
    const TuneKey key{(int)p, 2 + a.dagger};
    int id = -1;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        auto it = c->chosen.find(key);
        if (it != c->chosen.end()) id = it->second;
    }
    if (c->force_variant >= 0) id = c->force_variant;
    if (id < 0) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        if (cap != cudaStreamCaptureStatusNone) return fail(CD_ERR_INVALID, "tune apply_chain before capturing it");
        // tune: time a short chain of every fine-grained variant that fits co-resident, on
        // scratch fields (a chain writes both of its buffers; the caller's x must survive)
        const size_t fb = coarse_field_bytes(c, p);
        void *scratch = nullptr;
        CUDA_TRY(cudaMallocAsync(&scratch, 2 * fb, s), "cudaMallocAsync(tune scratch)");
        CUDA_TRY(cudaMemsetAsync(scratch, 0, 2 * fb, s), "cudaMemsetAsync");
        ApplyArgs ta = a;
        ta.in = scratch;
        ta.out = static_cast<unsigned char *>(scratch) + fb;
        cudaEvent_t e0, e1;
        CUDA_TRY(cudaEventCreate(&e0), "event");
        CUDA_TRY(cudaEventCreate(&e1), "event");
        float best = 1e30f;
        std::vector<int> cands{LLWARP_CHAIN_ID, CPUSH_CHAIN_ID, CLUSTER_CHAIN_ID};
        for (int i = 0; i < kNumLLReg; i++) cands.push_back(LLREG_CHAIN_ID0 + 1 + i);
        for (int v = 0; v < variant_count(p, c->nvec); v++) {
            cands.push_back(LL_CHAIN_ID0 + v);
            cands.push_back(v);
        }
        auto timeit = [&](int v, int trial) -> float {
            if (chain_launch(c, p, v, ta, 2, s) != cudaSuccess) {
                cudaGetLastError();
                return -1.f;
            }
            cudaEventRecord(e0, s);
            cudaError_t e = chain_launch(c, p, v, ta, trial, s);
            cudaEventRecord(e1, s);
            if (e != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess) {
                cudaGetLastError();
                return -1.f;
            }
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            return ms;
        };
        // pass 1: 64 applies of every candidate; pass 2: the three fastest, 512 applies, 3 rounds
        std::vector<std::pair<float, int>> t1;
        for (int v : cands) {
            const float ms = timeit(v, 64);
            if (ms >= 0.f) t1.emplace_back(ms, v);
        }
        std::sort(t1.begin(), t1.end());
        if (t1.size() > 3) t1.resize(3);
        std::vector<float> t2(t1.size(), 1e30f);
        for (int round = 0; round < 3; round++)
            for (size_t i = 0; i < t1.size(); i++) {
                const float ms = timeit(t1[i].second, 512);
                if (ms >= 0.f) t2[i] = std::min(t2[i], ms);
            }
        for (size_t i = 0; i < t1.size(); i++)
            if (t2[i] < best) best = t2[i], id = t1[i].second;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFreeAsync(scratch, s);
        if (id < 0) return fail(CD_ERR_UNSUPPORTED, "no chain variant fits this lattice co-resident");
        std::lock_guard<std::mutex> lk(c->mu);
        c->chosen[key] = id;
    }
    const char *tf = getenv("CD_CHAIN_TRACE");   // diagnostic only: clock64 events of CTA 0 (LL-register chain)
    if (tf && ((id > LLREG_CHAIN_ID0 && id < LLREG_CHAIN_ID0 + 100) || id == CPUSH_CHAIN_ID))
        CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&a.trace), 40 * 1024 * sizeof(long long), s), "trace");
    if (a.trace) CUDA_TRY(cudaMemsetAsync(a.trace, 0, 40 * 1024 * sizeof(long long), s), "trace");
    cudaError_t e = chain_launch(c, p, id, a, n, s);
    if (a.trace) {
        std::vector<long long> h(40 * 1024);
        cudaMemcpyAsync(h.data(), a.trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        cudaFreeAsync(a.trace, s);
        if (FILE *f = fopen(tf, "wb")) {
            fwrite(h.data(), sizeof(long long), h.size(), f);
            fclose(f);
        }
    }
    if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(CD_ERR_UNSUPPORTED, "chain variant does not fit co-resident / not a chain variant");
    }
    CUDA_TRY(e, "chain launch");
    return CD_OK;
    API_END
}

int coarse_halo_pack(cd_context *c, const cd_field *in, void *dst, int dst_on_device, size_t *bytes, void *stream)
{
    API_BEGIN
    if (!c || !in || !bytes) return fail(CD_ERR_INVALID, "ctx/in/bytes is NULL");
    CTX_GUARD(c);
    if (in->ctx != c) return fail(CD_ERR_MISMATCH, "field from another context");
    if (c->kg.split == 0) {
        *bytes = 0;
        return CD_OK;
    }
    const size_t n = halo_bytes(c, in->prec);
    *bytes = n;
    if (!dst) return CD_OK;
    cudaStream_t s = S(stream);
    KGeom g = halo_geom(c, in->prec);
    const cd_halo_plan pl = ctx_plan(c, in->prec);
    PackDst pd{};
    for (int mu = 0; mu < 4; mu++)
        for (int b = 0; b < 2; b++) pd.dst[mu][b] = static_cast<unsigned char *>(c->send_buf) + pl.block_offset[mu][b];
    CUDA_TRY(launch_pack(in->prec, c->nvec, in->base, pd, g, s), "halo pack");
    CUDA_TRY(cudaMemcpyAsync(dst, c->send_buf, n, dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(pack)");
    if (!dst_on_device) CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return CD_OK;
    API_END
}

int coarse_halo_exchange(cd_context *c, const cd_field *in, void *dst, int dst_on_device, size_t *bytes, void *stream)
{
    API_BEGIN
    if (!c || !in || !bytes) return fail(CD_ERR_INVALID, "ctx/in/bytes is NULL");
    if (in->ctx != c) return fail(CD_ERR_MISMATCH, "field from another context");
    if (in->nrhs != 1 || in->parity >= 0) return fail(CD_ERR_INVALID, "needs an ordinary full-lattice field");
    CTX_GUARD(c);
    if (c->kg.split == 0) {
        *bytes = 0;
        return CD_OK;
    }
    std::string err;
    int r = transport_check(c, err);
    if (r != CD_OK) return fail(r, err);
    c->applied = true;
    cudaStream_t s = S(stream);
    const cd_halo_plan pl = ctx_plan(c, in->prec);
    *bytes = (size_t)pl.total_bytes;
    HaloX x;
    r = halo_begin(c, pl, &x, err);
    if (r != CD_OK) return fail(r, err);
    CUDA_TRY(launch_pack(in->prec, c->nvec, in->base, x.pd, halo_geom(c, in->prec), s), "halo pack");
    r = halo_post(c, pl, x, s, err);
    if (r != CD_OK) return fail(r, err);
    r = halo_finish(c, x, s, err);
    if (r != CD_OK) return fail(r, err);
    if (dst) {
        CUDA_TRY(cudaMemcpyAsync(dst, x.recv, *bytes, dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(recv)");
        if (!dst_on_device) CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
    return CD_OK;
    API_END
}

int cd_context_peer_handle(cd_context *c, uint8_t out_handle[64])
{
    API_BEGIN
    if (!c || !out_handle) return fail(CD_ERR_INVALID, "ctx/out is NULL");
    CTX_GUARD(c);
    std::string err;
    const size_t slot = std::max(halo_bytes(c, CD_FP32), halo_bytes(c, CD_FP16));
    int r = peer_window_export(c, slot, out_handle, err);
    if (r != CD_OK) return fail(r, err);
    return CD_OK;
    API_END
}

int cd_context_peer_connect(cd_context *c, const uint8_t *handles, int nranks)
{
    API_BEGIN
    if (!c || !handles) return fail(CD_ERR_INVALID, "ctx/handles is NULL");
    CTX_GUARD(c);
    std::string err;
    int r = peer_connect(c, handles, nranks, err);
    if (r != CD_OK) return fail(r, err);
    c->chosen.clear();
    return CD_OK;
    API_END
}

int cd_halo_plan_create(const cd_geometry *geom, int nranks, int rank, cd_precision prec, int32_t self_mask,
                        cd_halo_plan *out)
{
    API_BEGIN
    if (!out) return fail(CD_ERR_INVALID, "out is NULL");
    int r = check_geometry(geom, nranks, rank);
    if (r != CD_OK) return r;
    if (prec != CD_FP32 && prec != CD_FP16) return fail(CD_ERR_INVALID, "bad precision");
    if (self_mask < 0 || self_mask > 15) return fail(CD_ERR_INVALID, "self_mask must be in [0, 15]");
    for (int mu = 0; mu < 4; mu++)
        if (((self_mask >> mu) & 1) && geom->proc_grid[mu] != 1)
            return fail(CD_ERR_INVALID, "self_mask dims must have proc_grid == 1");
    make_plan(geom, rank, prec, self_mask, out);
    return CD_OK;
    API_END
}

int cd_flush_l2(cd_context *c, size_t bytes, void *stream)
{
    API_BEGIN
    if (!c) return fail(CD_ERR_INVALID, "ctx is NULL");
    CTX_GUARD(c);
    static void *buf = nullptr;
    static size_t cap = 0;
    if (bytes > cap) {
        if (buf) cudaFree(buf);
        buf = nullptr;
        cap = 0;
        CUDA_TRY(cudaMalloc(&buf, bytes), "cudaMalloc(flush)");
        cap = bytes;
    }
    CUDA_TRY(launch_flush(buf, bytes, S(stream)), "flush kernel");
    return CD_OK;
    API_END
}

// ------------------------------------------------------------------ transfer operators (NEXT-4)
int coarse_transfer_create(cd_context *c, const cd_transfer_desc *d, const void *basis, int src_on_device,
                           cd_host_dtype dt, void *stream, cd_transfer **out)
{
    API_BEGIN
    if (!c || !d || !basis || !out) return fail(CD_ERR_INVALID, "ctx/desc/basis/out is NULL");
    CTX_GUARD(c);
    if (dt != CD_C64 && dt != CD_C128) return fail(CD_ERR_INVALID, "bad dtype");
    if (d->nspin != 2 && d->nspin != 4) return fail(CD_ERR_UNSUPPORTED, "nspin must be 2 or 4");
    if (d->ncolor < 1 || d->ncolor > 256) return fail(CD_ERR_INVALID, "ncolor must be in [1, 256]");
    TGeom t{};
    t.c = c->kg;
    t.Bvol = 1;
    int64_t Vf = 1;
    for (int mu = 0; mu < 4; mu++) {
        if (d->block[mu] < 1) return fail(CD_ERR_INVALID, "block dims must be >= 1");
        t.B[mu] = d->block[mu];
        t.Lf[mu] = c->local[mu] * d->block[mu];
        t.Bvol *= d->block[mu];
        Vf *= t.Lf[mu];
    }
    t.nf = d->nspin * d->ncolor;
    if (Vf * t.nf * c->nvec >= ((int64_t)1 << 40) || Vf >= ((int64_t)1 << 31))
        return fail(CD_ERR_INVALID, "fine lattice too large");
    t.Vf = (int)Vf;
    const size_t n = (size_t)Vf * t.nf * c->nvec;
    cudaStream_t s = S(stream);
    void *W = nullptr;
    CUDA_TRY(cudaMalloc(&W, n * 8), "cudaMalloc(basis)");
    cudaError_t e = cudaSuccess;
    if (dt == CD_C64) {
        e = cudaMemcpyAsync(W, basis, n * 8, src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
    } else {
        const void *src = basis;
        void *stage = nullptr;
        if (!src_on_device) {
            e = cudaMallocAsync(&stage, n * 16, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(stage, basis, n * 16, cudaMemcpyHostToDevice, s);
            src = stage;
        }
        if (e == cudaSuccess) e = launch_c128_to_c64(src, W, (int64_t)n, s);
        if (stage) cudaFreeAsync(stage, s);
    }
    if (e != cudaSuccess) {
        cudaFree(W);
        return cuda_fail(e, "basis upload");
    }
    *out = new cd_transfer{c, {d->block[0], d->block[1], d->block[2], d->block[3]}, d->nspin, d->ncolor, W, n * 8, t};
    return CD_OK;
    API_END
}

int coarse_transfer_free(cd_transfer *t)
{
    API_BEGIN
    if (!t) return fail(CD_ERR_INVALID, "transfer is NULL");
    cudaFree(t->W);
    delete t;
    return CD_OK;
    API_END
}

size_t coarse_transfer_fine_bytes(const cd_transfer *t)
{
    return t ? (size_t)t->tg.Vf * t->tg.nf * 8 : 0;
}

int coarse_transfer_read_basis(const cd_transfer *t, void *dst, int dst_on_device, void *stream)
{
    API_BEGIN
    if (!t || !dst) return fail(CD_ERR_INVALID, "transfer/dst is NULL");
    CTX_GUARD(t->ctx);
    CUDA_TRY(cudaMemcpyAsync(dst, t->W, t->wbytes, dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             S(stream)),
             "cudaMemcpyAsync(basis)");
    if (!dst_on_device) CUDA_TRY(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize");
    return CD_OK;
    API_END
}

int coarse_transfer_orthonormalise(cd_transfer *t, void *stream)
{
    API_BEGIN
    if (!t) return fail(CD_ERR_INVALID, "transfer is NULL");
    CTX_GUARD(t->ctx);
    if ((int64_t)t->tg.Bvol * (t->tg.nf / 2) < t->ctx->nvec)
        return fail(CD_ERR_INVALID, "aggregate has fewer rows per chirality than Nvec columns");
    if (t->tg.Bvol * (int64_t)sizeof(int) > 200 * 1024) return fail(CD_ERR_UNSUPPORTED, "aggregate too large");
    cudaStream_t s = S(stream);
    DevBuf fb;
    CUDA_TRY(cudaMalloc(&fb.p, sizeof(int)), "cudaMalloc");
    int *flag = static_cast<int *>(fb.p);
    CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s), "cudaMemsetAsync");
    CUDA_TRY(launch_orthonormalise(t->ctx->nvec, t->W, t->tg, flag, s), "orthonormalise kernel");
    int h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    if (h) return fail(CD_ERR_INVALID, "rank-deficient aggregate block (DESIGN.md R21)");
    return CD_OK;
    API_END
}

static int check_transfer(const cd_transfer *t, const cd_field *f, const void *fine)
{
    if (!t || !f || !fine) return fail(CD_ERR_INVALID, "transfer/field/fine is NULL");
    if (f->ctx != t->ctx) return fail(CD_ERR_MISMATCH, "field from another context");
    if (f->nrhs != 1 || f->parity >= 0) return fail(CD_ERR_INVALID, "needs an ordinary full-lattice coarse field");
    return CD_OK;
}

int coarse_restrict(const cd_transfer *t, cd_field *coarse_out, const void *fine_in, void *stream)
{
    API_BEGIN
    int r = check_transfer(t, coarse_out, fine_in);
    if (r != CD_OK) return r;
    const int cl = restrict_cluster_size(t->tg, t->ctx->num_sms);
    CUDA_TRY(launch_restrict(coarse_out->prec, t->ctx->nvec, cl, t->W, fine_in, coarse_out->base, t->tg, S(stream)),
             "restrict kernel");
    return CD_OK;
    API_END
}

int coarse_prolong(const cd_transfer *t, void *fine_out, const cd_field *coarse_in, void *stream)
{
    API_BEGIN
    int r = check_transfer(t, coarse_in, fine_out);
    if (r != CD_OK) return r;
    CUDA_TRY(launch_prolong(coarse_in->prec, t->ctx->nvec, t->W, coarse_in->base, fine_out, t->tg, S(stream)),
             "prolong kernel");
    return CD_OK;
    API_END
}

}  // extern "C"
