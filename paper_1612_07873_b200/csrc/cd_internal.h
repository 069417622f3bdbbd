// cd_internal.h -- host runtime structures of the coarse-Dslash library (not part of the ABI).
//
// Internal stored records (DESIGN.md §5 "Data layout in HBM"):
//   fp32 vector record  : N float2                              (8N bytes)
//   fp16 vector record  : N half2 {re,im} + float scale + 12 B  (4N + 16 bytes)
//   fp32 matrix record  : N*N float2, row-major                 (8N^2 bytes)
//   fp16 matrix record  : N*N half2 + float scale + 12 B        (4N^2 + 16 bytes)
//   field  = V records, site-major (canonical site order)
//   links  = V * 9 matrix records, [site][k]   -> one site's 9 matrices are contiguous
// Every record is a multiple of 16 bytes, so every record can be moved by one
// cp.async.bulk (TMA 1-D) and read with 128-bit loads.
#pragma once

#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>
#include <map>
#include <mutex>

#include "../../include/coarse_dslash.h"

namespace cd {

inline size_t vec_rec_bytes(int N, cd_precision p) { return p == CD_FP32 ? size_t(8) * N : size_t(4) * N + 16; }
inline size_t mat_rec_bytes(int N, cd_precision p) { return p == CD_FP32 ? size_t(8) * N * N : size_t(4) * N * N + 16; }
inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Integer division by a run-time constant via a multiply-high (the "integer division magic
// numbers computed on the host" the paper proposes for the index decode).
// Valid for 0 <= n < 2^31, 1 <= d < 2^31:  q = (umulhi(n, m) + n) >> s.
struct FastDiv {
    uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d)
{
    FastDiv f{d, 0, 0};
    uint32_t s = 0;
    while ((uint64_t(1) << s) < d) s++;
    f.s = s;
    f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1);
    return f;
}
inline uint32_t fastdiv_host(uint32_t n, const FastDiv &f)
{
    uint64_t hi = (uint64_t(n) * f.m) >> 32;
    return uint32_t((hi + n) >> f.s);
}

// Kernel-visible geometry of the local lattice + halo description.
struct KGeom {
    int L[4];
    int V;
    FastDiv fd[3];          // divisions by L0, L1, L2 for the site decode
    int split;              // bit mu: dim mu goes through the halo path
    // halo wire format (R13): for split dim mu, block A then block B,
    // each F[mu] payload records of prec_rec bytes then (fp16) F[mu] float scales.
    int64_t blk_off[4][2];  // byte offset of block (mu, A/B) in the send / recv buffer
    int F[4];               // face sites of dim mu
};

// Transfer-operator geometry: fine lattice = coarse local lattice x block.
struct TGeom {
    KGeom c;     // coarse local lattice
    int B[4];    // aggregate (block) dims
    int Bvol;    // fine sites per aggregate
    int Lf[4];   // fine local dims
    int Vf;      // fine local volume
    int nf;      // fine dofs per site = Ns * Nc
};

struct Comm;  // comm.cpp

// Halo transports (CD_OPT_TRANSPORT).
enum Transport { TR_AUTO = 0, TR_NCCL = 1, TR_PEER = 2, TR_COPY = 3 };

// Peer window (TR_PEER): one cudaMalloc per rank, exported with CUDA IPC and mapped by the
// neighbours.  Header: arrival counters [mu][blk] (u64), padded to kWinHeader; then two
// receive slots of win_slot bytes (exchange e uses slot e % 2).
constexpr size_t kWinHeader = 4096;
constexpr int kPutCtas = 16;   // CTAs per (mu, blk) of every signalling kernel: +16 per block per exchange

// Where the halo pack kernel writes block (mu, blk) (dst = block base incl. its offset) and,
// for the peer transport, the receiver's arrival counter it bumps once per CTA (nullptr: none).
struct PackDst {
    unsigned char *dst[4][2];
    unsigned long long *flag[4][2];
};

// Receiver side of one peer exchange: spin (acquire, system scope) until every block in `mask`
// (bit 2mu+blk) has counter >= target; on timeout set *err and return (no hang).
struct PeerWait {
    const unsigned long long *flag;
    unsigned mask;
    unsigned long long target;
    int *err;
    unsigned long long timeout_ns;
};

struct TuneKey {
    int prec, dagger;
    bool operator<(const TuneKey &o) const { return prec != o.prec ? prec < o.prec : dagger < o.dagger; }
};

}  // namespace cd

struct cd_context {
    cd_geometry geom{};
    int device = 0, nranks = 1, rank = 0;
    int coords[4] = {0, 0, 0, 0};
    int local[4] = {1, 1, 1, 1};
    int64_t V = 0;
    int N = 0, nvec = 0;
    int nbr_rank[4][2] = {};      // [mu][0] = rank at +mu, [mu][1] = rank at -mu
    cd::KGeom kg{};
    // halo resources (allocated lazily on first partitioned apply)
    void *send_buf = nullptr, *recv_buf = nullptr;
    size_t halo_cap = 0;
    float2 *face_scratch = nullptr;   // fp32 partial y for face sites [V][N]
    int *face_sites = nullptr;        // device list of face site indices
    int *interior_sites = nullptr;    // device list of the other sites (multi-RHS overlap)
    int n_interior = 0;
    void *mrhs_send = nullptr, *mrhs_recv = nullptr;   // multi-RHS halo buffers (lazy)
    size_t mrhs_cap = 0;
    int *pack_cnt = nullptr;          // fused split apply: pack-completion counter (zero between launches)
    int *work = nullptr;              // ring kernel ticket counters (4 slots x 2 ints, zero between
                                      // launches); applies on one context must be stream-ordered
    uint32_t seq = 0;                 // dslash launch sequence number
    float2 *ysplit = nullptr;         // fp16 row-split scratch [V][N]
    int *site_cnt = nullptr;          // fp16 row-split per-site counters [V]
    unsigned *chain_cnt = nullptr;    // chain kernel per-site counters [V] (monotonic)
    unsigned chain_base = 0;          // value every chain counter holds between chain calls
    void *llbuf = nullptr;            // LL chain buffers (allocated on first use, zeroed)
    unsigned ll_base = 0;             // LL chain epochs used so far
    int n_face = 0;
    bool halo_ready = false;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
    cd::Comm *comm = nullptr;
    // halo transport
    int transport = 0;                // CD_OPT_TRANSPORT
    int nccl_sm_reserve = 4;          // CD_OPT_NCCL_SM_RESERVE: SMs the interior leaves to NCCL (capped at 4 CTAs)
    unsigned char *win = nullptr;     // own peer window (kWinHeader + 2 slots)
    size_t win_slot = 0;
    unsigned char *peer_win[4][2] = {};   // window of the rank at +mu (dir 0) / -mu (dir 1)
    std::vector<void *> ipc_opened;   // IPC mappings to close
    bool peer_ready = false;
    uint64_t epoch = 0;               // peer exchanges issued so far (identical sequence on every rank)
    int *err_host = nullptr;          // host-mapped transport error word (peer wait timeouts)
    int *err_dev = nullptr;
    unsigned long long peer_timeout_ns = 60ull * 1000 * 1000 * 1000;
    // options
    int force_variant = -1;
    int tune = 1;
    int halo_self_mask = 0;
    int pdl = 1;
    int fuse_split = 1;               // CD_FUSE_SPLIT=0: peer-transport ring applies use the unfused path
    bool applied = false;
    int num_sms = 148;
    // tuning results per (prec, dagger)
    std::map<cd::TuneKey, int> chosen;
    std::mutex mu;
};

struct cd_field {
    cd_context *ctx;
    cd_precision prec;
    void *base;
    size_t bytes;
    bool owned;
    int nrhs;   // right-hand sides (records stored [site][rhs]); 1 for an ordinary field
    int parity; // -1: full lattice; 0 / 1: the V/2 even / odd sites in half-index order (s >> 1)
};

struct cd_links {
    cd_context *ctx;
    cd_precision prec;
    void *base;
    size_t bytes;
    int compressed;   // 1: tau3-hermitian compressed storage (X + 4 forward links per site)
    int eo;           // 1: even-odd prepared: base = even sites [V/2][9], aux = odd [V/2][8] (X^-1 L_k)
    void *aux;        // eo: odd-site records
    void *tbuf;       // eo: odd half-field scratch t_o (fp32)
    int64_t lhoff[4] = {0, 0, 0, 0};   // compressed + multi-rank: aux = link halo, dim mu's records at lhoff[mu]
    int split = 0;                     // compressed: the context's halo split mask when the link halo was built
};

struct cd_transfer {
    cd_context *ctx;
    int block[4];
    int nspin, ncolor;
    void *W;          // basis, fp32 complex [Vf][nf][Nvec]
    size_t wbytes;
    cd::TGeom tg;
};

namespace cd {

// ---- launchers implemented in .cu files (return cudaError_t of the launch)
struct ApplyArgs {
    const void *links;
    const void *in;
    void *out;
    float2 *scratch;       // face-site fp32 partials (halo mode) or nullptr
    const void *recv;      // halo receive buffer (halo kernel)
    const int *face_sites; // halo kernel site list
    int n_face;
    int *work;             // ring: 4 slots x {site tickets, finished CTAs} (reset by the last CTA)
    uint32_t seq;          // launch sequence number (ring ticket slot = seq % 4)
    float2 *ysplit;        // fp16 row-split fg: fp32 rows of a site [V][N] (L2 resident)
    int *site_cnt;         // fp16 row-split fg: per-site arrival counters (zero between launches)
    unsigned *chain_cnt;   // chain kernel: monotonic per-site completion counters
    void *llbuf;           // LL chain: 2 x V LL records (epoch-tagged payload words)
    int poll_ns;           // LL chain: __nanosleep between unsuccessful polls (0 = spin); LL-register: before the first poll
    int poll_d0;           // LL-register chain: first poll of an apply no earlier than this many cycles after its start
    int poll_d1;           // LL-register chain: cycles between unsuccessful polls
    KGeom g;
    int nvec;
    int dagger;
    int halo;              // 1: skip remote hops, face sites -> scratch
    const void *lhalo;     // compressed links, multi-rank: the -mu neighbours' x_mu = L-1 forward records
    int64_t lhoff[4];      // byte offset of dim mu's records in lhalo
    long long *trace;      // LL-register chain diagnostic (CD_CHAIN_TRACE): clock64 events of CTA 0
    // fused split apply (ring variants + peer transport): the ring kernel packs its
    // slice of the face records straight into the neighbours' windows in its prologue (the last
    // CTA to finish signals kPutCtas per block), takes interior sites before face sites, and its
    // producer reads a face site's remote records from this rank's window after an in-kernel
    // arrival wait -- one launch per apply, no halo-term kernel, no partials
    int fused;                           // 1: fused split apply (peer transport)
    PackDst pd;                          // pack destinations + the peers' arrival counters
    const unsigned long long *wflag;     // this rank's arrival counters [mu][blk]
    unsigned wmask;                      // blocks to wait for (bit 2mu+blk)
    unsigned long long wtarget;          // counter value of this exchange
    unsigned long long wtimeout;         // ns
    int *werr;                           // host-mapped error word (timeout)
    int *pack_cnt;                       // CTAs done with their pack slice (last one resets it)
    int rot;                             // ticket -> site rotation (T-only split: V / L3 puts the T faces last)
};

constexpr int CLUSTER_CHAIN_ID = 1000;   // apply_chain variant: whole lattice in one cluster
constexpr int CPUSH_CHAIN_ID = 4000;     // apply_chain variant: one cluster, DSMEM push (fp32, Nvec 24)
constexpr int LLWARP_CHAIN_ID = 5000;    // apply_chain variant: LL protocol, one warp per 4 rows (fp32)
constexpr int LL_CHAIN_ID0 = 2000;       // apply_chain variants 2000 + fg id: LL-protocol chain
constexpr int LLREG_CHAIN_ID0 = 3000;    // apply_chain variants 3001 + i: LL-register chain (fp32), i < kNumLLReg
constexpr int kNumLLReg = 6;

int variant_count(cd_precision p, int nvec);
const char *variant_name(cd_precision p, int nvec, int id);
bool variant_valid(cd_precision p, int nvec, int id, const KGeom &g);
int variant_heuristic(cd_precision p, int nvec, const KGeom &g, int num_sms);
cudaError_t launch_dslash(cd_precision p, int id, const ApplyArgs &a, cudaStream_t s, bool pdl, int num_sms);
cudaError_t launch_halo(cd_precision p, const ApplyArgs &a, cudaStream_t s);
cudaError_t launch_pack(cd_precision p, int nvec, const void *field, const PackDst &d, const KGeom &g, cudaStream_t s);
cudaError_t launch_peer_wait(const PeerWait &w, cudaStream_t s);

// bulk peer put of one chunk: for every block in `mask`, len[mu][blk] bytes from src[mu][blk] to
// d.dst[mu][blk], then bump d.flag[mu][blk] once per CTA (kPutCtas CTAs per block)
cudaError_t launch_peer_put(const unsigned char *const src[4][2], const int64_t len[4][2], unsigned mask,
                            const PackDst &d, cudaStream_t s);
cudaError_t launch_copy_blocks(const unsigned char *const src[4][2], unsigned char *const dst[4][2],
                               const int64_t len[4][2], unsigned mask, cudaStream_t s);

cudaError_t launch_import(cd_precision p, int nvec, int64_t nsites, const void *src, int src_c128, void *dst,
                          cudaStream_t s, int nrhs = 1);
cudaError_t launch_export(cd_precision p, int nvec, int64_t nsites, const void *src, void *dst, int dst_c128,
                          cudaStream_t s, int nrhs = 1);
cudaError_t launch_links_convert(cd_precision p, int nvec, int64_t nmats, const void *src, int src_c128, void *dst,
                                 cudaStream_t s, int64_t mat0);
cudaError_t launch_links_generate(cd_precision p, int nvec, const cd_context *ctx, int kind, uint64_t seed,
                                  int scale_log2, void *dst, cudaStream_t s);
cudaError_t launch_field_generate(cd_precision p, int nvec, const cd_context *ctx, uint64_t seed, uint32_t tag,
                                  int scale_log2, void *dst, cudaStream_t s, int nrhs = 1);
cudaError_t launch_eo_prepare(int nvec, const void *full, void *even, void *odd, const KGeom &g, int *singular,
                              cudaStream_t s);
struct EoApply {              // one even-odd Schur apply (coarse_dslash_apply_eo)
    const void *even, *odd;   // prepared links: even [V/2][9], odd [V/2][8]
    const void *in_e;
    void *t_o, *out_e;
    KGeom g;                  // halo geometry when split != 0
    int dagger;
    cudaStream_t s;
    bool pdl;
    // multi-rank (split != 0)
    int halo;
    cudaStream_t comm_stream;
    cudaEvent_t ev_in, ev_halo;
    float2 *scratch;
    const int *face_sites;
    int n_face;
    // one halo exchange per stage: begin() gives the pack destinations and the receive buffer,
    // post() starts the transfer on comm_stream after the pack, finish() orders the arrival
    // before the halo kernel on s (peer transport: the wait kernel)
    cudaError_t (*begin)(void *, PackDst *, const void **recv);
    cudaError_t (*post)(void *);
    cudaError_t (*finish)(void *);
    void *exchange_arg;
};
cudaError_t launch_eo_apply(int nvec, const EoApply &e);
cudaError_t launch_fgh(cd_precision p, const ApplyArgs &a, cudaStream_t s, bool pdl);
cudaError_t launch_compress(cd_precision p, int nv, const void *full, void *comp, int64_t nsites, cudaStream_t s);
cudaError_t launch_hermdev(cd_precision p, int nv, const void *full, const KGeom &g, float *dev, cudaStream_t s,
                           const void *lhalo = nullptr, const int64_t *lhoff = nullptr);
cudaError_t launch_fgh_halo(cd_precision p, const ApplyArgs &a, cudaStream_t s);
cudaError_t launch_lhalo_pack(cd_precision p, int nv, const void *comp, void *send, const KGeom &g, const int64_t *off,
                              cudaStream_t s);
// multi-RHS halo: receive buffer in the tensor-core wire layout (per split dim: block A = the
// x_mu = L-1 face records for the +mu neighbour, block B = the x_mu = 0 face, each [face f][rb])
struct MrhsHalo {
    const void *recv;        // nullptr: single rank (no remote hops)
    int64_t off[4][2];       // byte offset of block (mu, A/B)
};
cudaError_t launch_mrhs(int nvec, const void *links, const void *in, void *out, const KGeom &g, int nrhs, int dagger,
                        cudaStream_t s, int num_sms, const int *sites = nullptr, int nsites = 0,
                        const MrhsHalo *halo = nullptr);
cudaError_t launch_mrhs_pack(int nvec, const void *field, void *send, const KGeom &g, int nrhs, const MrhsHalo &offs,
                             cudaStream_t s);
cudaError_t launch_flush(void *buf, size_t bytes, cudaStream_t s);
int restrict_cluster_size(const TGeom &t, int num_sms);
cudaError_t launch_restrict(cd_precision pc, int nvec, int cl, const void *W, const void *vf, void *vc, const TGeom &t,
                            cudaStream_t s);
cudaError_t launch_prolong(cd_precision pc, int nvec, const void *W, const void *vc, void *vf, const TGeom &t,
                           cudaStream_t s);
cudaError_t launch_orthonormalise(int nvec, void *W, const TGeom &t, int *fail, cudaStream_t s);
cudaError_t launch_c128_to_c64(const void *in, void *out, int64_t n, cudaStream_t s);

void count_launch(int n = 1);

}  // namespace cd
