/*
 * coarse_dslash.h -- C ABI of the B200-native coarse-grid Dirac operator.
 *
 * The operator (§3.4 Eq. 3, read as DESIGN.md R1-R10):
 *
 *     y(x) = X(x) v(x) + sum_{mu=0..3} [ L_{2mu}(x) v(x+mu) + L_{2mu+1}(x) v(x-mu) ]
 *
 * on a periodic 4-D coarse lattice; every L_k(x) is a dense N x N complex matrix with
 * N = 2*Nvec (coarse spin 2 x Nvec colours).  The dagger is
 * tau3 D tau3 (R5; PAPER.md:121 footnote 1).
 *
 * CANONICAL LAYOUTS (what import/export/upload read and write):
 *   site   s = ((x3*L2 + x2)*L1 + x1)*L0 + x0     x0 fastest (Listing 2)
 *   dof    i = sigma*Nvec + c                     spin slower (Listing 3)
 *   hop    k = 2*mu + dir; dir 0 -> +mu, dir 1 -> -mu; k = 8 -> X   (§6.3)
 *   vector   v[s][i]          complex, interleaved {re, im}
 *   links    L[s][k][i][j]    complex, row-major: y_i += L[i][j] v_j
 * With nranks > 1 every rank passes its LOCAL block (local dims = global / proc_grid),
 * indexed with local coordinates; rank r owns the block at grid coordinates
 * c = (r % P0, (r / P0) % P1, ...) (lexicographic like sites).
 *
 * STORAGE PRECISION (a run-time attribute of every field / link set):
 *   CD_FP32  fp32 payload.
 *   CD_FP16  IEEE binary16 payload normalised by an fp32 scale, one scale per site
 *            for vectors and one per (site, k) matrix for links (R12, the
 *            paper's "16-bit ... storage format" with a scale).
 *   Arithmetic is always fp32 (R11).
 *
 * CONVENTIONS
 *   - Every function returns a cd_status; on failure cd_last_error() gives a
 *     thread-local message.  No C++ exception and no abort() crosses this ABI.
 *   - Argument errors are detected synchronously and nothing is enqueued.
 *   - Data calls are asynchronous and stream-ordered on the caller's cudaStream_t
 *     (passed as void*; NULL = legacy default stream).  They never synchronise the
 *     host, except coarse_links_upload / *_read_stored from host memory, which return
 *     once the host source (destination) has been consumed (filled).
 *   - Asynchronous CUDA / NCCL faults surface at the next call that observes them.
 *   - Pointers are borrowed for the duration of the stream-ordered work only; the
 *     library never keeps a caller pointer except caller-provided field memory
 *     (coarse_field_alloc with device_mem != NULL), which stays caller-owned.
 *   - apply / apply_dagger are COLLECTIVE when nranks > 1: every rank calls them in
 *     the same order.  They are CUDA-graph capturable once the (volume, Nvec,
 *     precision, op, partition) key has been tuned (first call; or CD_TUNE=0).
 *   - SINGLE STREAM PER CONTEXT: all operator calls (apply, apply_dagger, apply_chain,
 *     apply_mrhs, apply_eo) on one context must be ordered on one stream (or on streams
 *     the caller orders with events).  The persistent kernels' work tickets and the halo
 *     transport's epochs are per-context sequence numbers; two concurrently running
 *     applies on one context would share them.  Use one context per stream instead.
 *   - Every entry point makes the context's device current for its duration and restores
 *     the caller's current device before returning.
 *   - Link objects have a kind: full (upload / generate), compressed
 *     (coarse_links_compress_hermitian) or even-odd (coarse_links_prepare_eo).  A call
 *     given a kind it does not support returns CD_ERR_INVALID without enqueuing work.
 */
#ifndef COARSE_DSLASH_H
#define COARSE_DSLASH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
    CD_OK = 0,
    CD_ERR_INVALID = -1,      /* bad argument (NULL, size, alias, range)               */
    CD_ERR_UNSUPPORTED = -2,  /* valid but not implemented (e.g. Nvec not in {24, 32}) */
    CD_ERR_OOM = -3,          /* device or host allocation failed                      */
    CD_ERR_CUDA = -4,         /* CUDA runtime error (message has cudaGetErrorString)   */
    CD_ERR_NCCL = -5,         /* NCCL error or libnccl.so.2 not loadable               */
    CD_ERR_MISMATCH = -6,     /* objects from different contexts / precisions          */
    CD_ERR_COMM = -7          /* peer halo transport fault (a neighbour's halo never arrived) */
} cd_status;

typedef enum { CD_FP32 = 0, CD_FP16 = 1 } cd_precision;    /* storage; arithmetic is fp32   */
typedef enum { CD_C64 = 0, CD_C128 = 1 } cd_host_dtype;     /* canonical complex element type */

typedef enum {                 /* synthetic link recipes   */
    CD_LINKS_GENERAL = 0,      /* L_k(x) = G(x, k)                                          */
    CD_LINKS_HERMITIAN = 1,    /* tau3-hermitian: L_{2mu+1}(x) = tau3 G(x-mu,2mu)^H tau3, X = (G+tau3 G^H tau3)/2 */
    CD_LINKS_TI_GENERAL = 2,   /* translation invariant (gsite := 0, tag 4)                 */
    CD_LINKS_TI_HERMITIAN = 3
} cd_links_kind;

typedef enum {
    CD_OPT_VARIANT = 0,        /* force a kernel variant id (>= 0), -1 = autotune (default) */
    CD_OPT_TUNE = 1,           /* 1 = autotune on first call of a key (default), 0 = heuristic */
    CD_OPT_HALO_SELF_MASK = 2, /* bit mu: route dim mu through the halo path even when P_mu = 1
                                  (self exchange; exercises pack/exchange/halo kernels on 1 GPU).
                                  Only valid before the first apply. */
    CD_OPT_PDL = 3,            /* 1 = programmatic dependent launch between kernels (default 1) */
    CD_OPT_TRANSPORT = 4,      /* halo transport:
                                    0 auto (default): peer if connected, else NCCL if the context
                                      has a communicator, else device copy (self exchanges only);
                                    1 NCCL: ncclSend/ncclRecv in one group on the comm stream; on a
                                      1-rank context this creates a 1-rank communicator and the self
                                      exchanges of CD_OPT_HALO_SELF_MASK go through NCCL self
                                      send/recv (the multi-rank group code on one GPU);
                                    2 peer: the halo pack kernel stores the faces straight into the
                                      neighbours' CUDA-IPC-mapped receive windows over NVLink and
                                      signals arrival counters; the receiver waits on the device
                                      (needs cd_context_peer_handle / cd_context_peer_connect); with
                                      a persistent (ring) variant the whole split apply is ONE
                                      launch that waits in-kernel for its neighbours -- one rank per
                                      GPU (or time-sliced processes); with several ranks sharing a
                                      GPU concurrently (MPS) set CD_FUSE_SPLIT=0;
                                    3 device copy (self exchanges only). */
    CD_OPT_NCCL_SM_RESERVE = 5,/* SMs the persistent interior kernel leaves free while an NCCL halo
                                  exchange is in flight (its kernels need SMs to progress); default 4
                                  (the library's communicators cap NCCL at CD_NCCL_MAX_CTAS = 4 CTAs) */
    CD_OPT_PEER_TIMEOUT_MS = 6 /* peer transport: give up waiting for a neighbour's halo after this
                                  long (the context then reports CD_ERR_COMM); default 60000 */
} cd_option;

typedef struct {
    int32_t global_dims[4];    /* L0..L3 (x0 fastest, x3 = T); each >= 1                     */
    int32_t nvec;              /* Nvec; N = 2*Nvec; supported: 24, 32 (CD_ERR_UNSUPPORTED)   */
    int32_t proc_grid[4];      /* P0..P3; prod == nranks; global_dims[mu] % P[mu] == 0       */
} cd_geometry;

typedef struct cd_context cd_context;
typedef struct cd_field cd_field;
typedef struct cd_links cd_links;

/* ------------------------------------------------------------------ context */

/* Library version string (static storage). */
const char *cd_version(void);

/* Thread-local message of the last failed call on this thread ("" if none). */
const char *cd_last_error(void);

/* NCCL unique id for a multi-rank context (rank 0 calls it and broadcasts the 128 bytes,
 * e.g. with torch.distributed).  CD_ERR_NCCL if libnccl.so.2 cannot be loaded. */
int cd_get_unique_id(uint8_t out_id[128]);

/* Create a context on CUDA device `device` for rank `rank` of `nranks`.
 * nccl_id: the 128-byte id from cd_get_unique_id (collective: all ranks call this
 * concurrently; NCCL transport), or NULL -- always for nranks == 1; for nranks > 1 the
 * context then has no NCCL communicator and must use the peer transport (connect it before
 * the first collective call).  Allocates halo/scratch buffers (device memory).
 * Errors: CD_ERR_INVALID (geometry), CD_ERR_UNSUPPORTED (nvec), CD_ERR_CUDA, CD_ERR_NCCL. */
int cd_context_create(const cd_geometry *geom, int device, int nranks, int rank, const uint8_t *nccl_id,
                      cd_context **out);

/* Destroy a context (synchronises its device; fields/links of it must be freed first).
 * Peer-connected contexts: every rank must have finished its collective calls (e.g. a
 * barrier) before any rank destroys its context -- a neighbour may still be writing into
 * this rank's window. */
int cd_context_destroy(cd_context *ctx);

/* Peer transport setup (collective, two steps).  cd_context_peer_handle
 * allocates this rank's receive window (zeroed, synchronously) and returns its 64-byte CUDA
 * IPC handle; the caller all-gathers the handles of all ranks (e.g. torch.distributed) into
 * handles[nranks][64] and passes them to cd_context_peer_connect, which maps the windows of
 * this rank's halo neighbours (NVLink / NVSwitch peers, or the same GPU for several processes
 * on one device).  Set CD_OPT_HALO_SELF_MASK before this.  After connect the transport option
 * "auto" selects the peer transport. */
int cd_context_peer_handle(cd_context *ctx, uint8_t out_handle[64]);
int cd_context_peer_connect(cd_context *ctx, const uint8_t *handles, int nranks);

/* Set a cd_option (see the enum).  CD_ERR_INVALID for an unknown option or bad value. */
int cd_context_set_option(cd_context *ctx, int option, int64_t value);

/* Local geometry: local dims (4 ints), local volume, rank grid coordinates (4 ints). */
int cd_context_local(const cd_context *ctx, int32_t local_dims[4], int64_t *local_volume,
                     int32_t grid_coords[4]);

/* Number of kernel variants for a precision, and the name of variant `id`
 * (static storage; NULL if out of range). */
int cd_variant_count(const cd_context *ctx, cd_precision prec);
const char *cd_variant_name(const cd_context *ctx, cd_precision prec, int id);

/* Variant chosen for (prec, dagger) by the tuner / heuristic for this context's geometry
 * (-1 if that key has not been resolved yet).  dagger = 2 / 3 query coarse_dslash_apply_chain's
 * choice for D / D^dagger (ids: fg variant = counter chain, 1000 = cluster chain, 2000 + fg
 * variant = LL chain, 3001 + i = LL-register chain, 4000 = cluster push chain, 5000 = LL-warp
 * chain). */
int cd_context_chosen_variant(const cd_context *ctx, cd_precision prec, int dagger);

/* Total kernels launched by this process through this library (for launch accounting). */
uint64_t cd_launch_count(void);

/* ------------------------------------------------------------------ fields */

/* Device bytes needed for one field of this context's local volume in `prec`
 * (internal stored representation; 256-byte aligned allocation unit). */
size_t coarse_field_bytes(const cd_context *ctx, cd_precision prec);

/* Create a field.  device_mem == NULL: the library allocates (cudaMalloc) and frees it.
 * Else device_mem (>= 256-byte aligned, >= coarse_field_bytes) is caller-owned and must
 * outlive the field.  Contents are undefined until imported / generated / computed. */
int coarse_field_alloc(cd_context *ctx, cd_precision prec, void *device_mem, size_t bytes, cd_field **out);

/* Multi right-hand-side fields (the paper's multi-RHS MG).
 * fp32: nrhs records stored [site][rhs].  fp16 with nrhs > 1: the tensor-core layout (DESIGN.md
 * R22), blocks of 128 right-hand sides per site [site][block][K chunk][rhs][16 B] + one fp32 scale
 * per (site, block) -- nrhs must be a multiple of 128 (bytes query returns 0, alloc
 * CD_ERR_UNSUPPORTED otherwise).  import / export / generate work on them with the canonical
 * layout [rhs][site][i] (each rhs an ordinary canonical vector; generate gives rhs r the tag
 * tag + r); read_stored returns the blocks as stored.  Only coarse_dslash_apply_mrhs operates on
 * them. */
size_t coarse_field_bytes_mrhs(const cd_context *ctx, cd_precision prec, int nrhs);
int coarse_field_alloc_mrhs(cd_context *ctx, cd_precision prec, int nrhs, void *device_mem, size_t bytes,
                            cd_field **out);

/* Free a field handle (and its memory iff library-owned). */
int coarse_field_free(cd_field *f);

/* Import the canonical LOCAL vector v[s][i] (V_local * N complex of `dtype`) from host
 * (src_on_device = 0; pinned memory gives an asynchronous copy) or device memory.
 * fp16 fields quantise per site (R12).  stream-ordered. */
int coarse_field_import(cd_field *f, const void *src, int src_on_device, cd_host_dtype dtype, void *stream);

/* Export the field as a canonical LOCAL vector (fp16: dequantised x = float(q) * s). */
int coarse_field_export(const cd_field *f, void *dst, int dst_on_device, cd_host_dtype dtype, void *stream);

/* Fill with the synthetic vector of seed/tag over GLOBAL site indices,
 * values scaled by 2^scale_log2.  fp16 fields are quantised as by import. */
int coarse_field_generate(cd_field *f, uint64_t seed, uint32_t tag, int32_t scale_log2, void *stream);

/* Raw stored representation, for bit-exact layout checks: canonical-order payload
 * (V * N complex of float (fp32) or binary16 (fp16)) followed, for fp16, by V float
 * scales.  *_stored_bytes gives the size.  read copies to host or device memory. */
size_t coarse_field_stored_bytes(const cd_field *f);
int coarse_field_read_stored(const cd_field *f, void *dst, int dst_on_device, void *stream);

/* ------------------------------------------------------------------ links */

/* Upload the canonical LOCAL link block L[s][k][i][j] (V_local * 9 * N * N complex of
 * `dtype`) from host or device memory into a new, immutable links object in `prec`
 * (fp16: quantised per (s, k) matrix, R12).  Host sources are staged through
 * a bounded device buffer; the call returns when the source has been consumed. */
int coarse_links_upload(cd_context *ctx, cd_precision prec, const void *links, int src_on_device,
                        cd_host_dtype dtype, void *stream, cd_links **out);

/* Generate a synthetic links object on the device (recipe `kind`, GLOBAL indices, so the
 * operator is the same for every partition), values scaled by 2^scale_log2. */
int coarse_links_generate(cd_context *ctx, cd_precision prec, int kind, uint64_t seed, int32_t scale_log2,
                          void *stream, cd_links **out);

/* Raw stored links: canonical payload (V*9*N*N complex float / binary16) then, for fp16,
 * V*9 float scales. */
size_t coarse_links_stored_bytes(const cd_links *l);
int coarse_links_read_stored(const cd_links *l, void *dst, int dst_on_device, void *stream);

int coarse_links_free(cd_links *l);

/* Hermiticity-compressed links: for tau3-hermitian operators -- every Galerkin
 * coarse operator with chirality-preserving aggregation, PAPER.md:121 fn. 1 -- the backward links
 * are L_{2mu+1}(x) = tau3 L_{2mu}(x-mu)^H tau3, so only X and the four forward links are stored
 * (5 of 9 matrices per site; the apply reads the neighbour's forward link transposed).  Creates a
 * new links object from `full`; if max_dev != NULL it also measures (host sync) the largest
 * deviation |L_{2mu+1}(x) - tau3 L_{2mu}(x-mu)^H tau3| (on the dequantised values for fp16) so the
 * caller can decide whether the compression is exact.  fp32 or fp16.  On a multi-rank context this
 * call is collective: it performs a one-time link halo exchange (each rank sends the forward
 * records of its x_mu = L_mu - 1 faces to the +mu neighbour) used by the backward hops of the
 * x_mu = 0 sites; applies with the result are collective like coarse_dslash_apply. */
int coarse_links_compress_hermitian(const cd_links *full, double *max_dev, void *stream, cd_links **out);

/* ------------------------------------------------------------------ operator */

/* out = D in  (Eq. 3).  in, out, links: same context and precision (else CD_ERR_MISMATCH);
 * out must not alias in (CD_ERR_INVALID).  Collective for nranks > 1 (halo exchange of
 * `in` over NCCL, overlapped with the interior).  The first call for a key autotunes
 * (several trial launches on `stream`, excluded from any timing). */
int coarse_dslash_apply(const cd_links *links, cd_field *out, const cd_field *in, void *stream);

/* out = tau3 D tau3 in  (= D^H in for tau3-hermitian links; R5). */
int coarse_dslash_apply_dagger(const cd_links *links, cd_field *out, const cd_field *in, void *stream);

/* n chained applies in ONE persistent kernel (latency regime: the coarsest grid, where the
 * operator is applied over and over): for t = 0..n-1, t even: y = D x, t odd: x = D y (with
 * dagger != 0: the tau3 dagger).  The result of the last apply is in y for odd n, in x for
 * even n.  CTAs keep their link rows on chip for all n applies and synchronise point to point
 * (per-site counters) instead of through kernel boundaries (the 2^4 lattice is
 * latency bound).  Single-rank contexts only; the first call per (precision, dagger) tunes
 * (host sync).  CD_ERR_UNSUPPORTED if the decomposition does not fit co-resident on the GPU
 * (use coarse_dslash_apply for large lattices). */
int coarse_dslash_apply_chain(const cd_links *links, cd_field *x, cd_field *y, int n, int dagger, void *stream);

/* out_r = D in_r (dagger: tau3 D tau3 in_r) for every right-hand side r of two multi-RHS fields
 * with the same nrhs (a multiple of 128), on the tcgen05 tensor cores: per site one
 * 128 x 2N x (9 * 2N) fp16 x fp16 -> fp32 GEMM accumulated in TMEM (the links are read once
 * for 128 right-hand sides); persistent warp-specialised kernel (TMA ring, tcgen05.mma, TMEM
 * double buffer).  fp16 storage only (CD_ERR_UNSUPPORTED otherwise).  Collective on multi-rank
 * contexts: face blocks are exchanged (NCCL) while the interior sites run. */
int coarse_dslash_apply_mrhs(const cd_links *links, cd_field *out, const cd_field *in, int dagger, void *stream);

/* ------------------------------------------------------------------ even-odd
 * Red-black preconditioning (§3.3; used on all MG levels): the Schur
 * complement on the even sites,  M_ee v_e = X_e v_e - D_eo X_o^{-1} D_oe v_e,  site parity
 * (x0+x1+x2+x3) mod 2.  Needs every LOCAL L_mu even; fp32 storage.  Multi-rank contexts: each
 * stage packs its input's face sites, exchanges them (NCCL, same wire format as the full
 * operator) overlapped with the interior kernel, then adds the remote hops (collective).
 * Parity fields hold the V/2 sites of one parity in half-index order h = s >> 1 (canonical
 * import/export layout [V/2][N]). */
size_t coarse_field_bytes_parity(const cd_context *ctx, cd_precision prec);
int coarse_field_alloc_parity(cd_context *ctx, cd_precision prec, int parity, void *device_mem, size_t bytes,
                              cd_field **out);

/* Setup: X_o^{-1} on every odd site (fp64 Gauss-Jordan with partial pivoting) and
 * X_o^{-1} L_k(o) for its 8 hops, plus the even sites' 9 matrices; host-synchronous (returns
 * CD_ERR_INVALID if some X_o is singular).  The result is a new links object for
 * coarse_dslash_apply_eo only. */
int coarse_links_prepare_eo(const cd_links *full, void *stream, cd_links **out);

/* out_e = M_ee in_e (dagger != 0: tau3 M_ee tau3 = M_ee^H for tau3-hermitian links); two
 * kernels: t_o = X_o^{-1} D_oe in_e, then out_e = X_e in_e - D_eo t_o. */
int coarse_dslash_apply_eo(const cd_links *eo_links, cd_field *out, const cd_field *in, int dagger, void *stream);

/* ------------------------------------------------------------------ transfer operators
 * Prolongator P and restrictor R = P^dagger between a fine lattice and this context's coarse
 * lattice (§3.4; kernels §6.6).  Aggregates are block[0..3]
 * hypercubes of fine sites; the fine local lattice is local_dims x block, so the operators
 * are rank-local (no communication) when the coarse lattice is partitioned.  A fine site carries
 * nspin x ncolor dofs r = s*ncolor + a; chirality 0 = spins s < nspin/2 (R20, P:121
 * fn. 1), so coarse dof i = chirality*Nvec + k.
 *   basis (the columns of P): complex [Vf][nspin][ncolor][Nvec], stored fp32 on the device;
 *   fine fields: DEVICE pointers to complex64 [Vf][nspin][ncolor] (caller-owned);
 *   coarse fields: ordinary fp32 or fp16 cd_field of the context. */
typedef struct cd_transfer cd_transfer;
typedef struct {
    int32_t block[4];   /* aggregate extent per dim (>= 1)                                  */
    int32_t nspin;      /* fine spins: 4 (Wilson-clover fine grid) or 2 (a coarse level)     */
    int32_t ncolor;     /* fine colours per spin: 3 (Wilson) or the finer level's Nvec       */
} cd_transfer_desc;

/* Upload the basis (host or device, c64 or c128) as given -- call coarse_transfer_orthonormalise
 * for setup step 3.  CD_ERR_UNSUPPORTED for nspin not in {2, 4}. */
int coarse_transfer_create(cd_context *ctx, const cd_transfer_desc *desc, const void *basis, int src_on_device,
                           cd_host_dtype dtype, void *stream, cd_transfer **out);
int coarse_transfer_free(cd_transfer *t);
/* Bytes of one fine field (complex64 [Vf][nspin][ncolor]). */
size_t coarse_transfer_fine_bytes(const cd_transfer *t);
/* Copy the stored basis (complex64 [Vf][nspin][ncolor][Nvec]) to dst; host-synchronous for host dst. */
int coarse_transfer_read_basis(const cd_transfer *t, void *dst, int dst_on_device, void *stream);
/* Setup step 3: per (aggregate, chirality) block, replace the basis rows by the Q of its QR
 * decomposition (modified Gram-Schmidt, fp64 sums), in place.  Host-synchronous; CD_ERR_INVALID if
 * a block is rank deficient (R21) or has fewer rows than Nvec. */
int coarse_transfer_orthonormalise(cd_transfer *t, void *stream);
/* coarse_out = P^dagger fine_in (restrictor): one CTA or thread-block cluster per
 * aggregate, deterministic reduction.  fine_in: device complex64 [Vf][nspin][ncolor]. */
int coarse_restrict(const cd_transfer *t, cd_field *coarse_out, const void *fine_in, void *stream);
/* fine_out = P coarse_in (prolongator: a gather per fine dof).  fine_out: device complex64. */
int coarse_prolong(const cd_transfer *t, void *fine_out, const cd_field *coarse_in, void *stream);

/* Halo send buffer of `in` in the canonical wire order (R13): packs on `stream`
 * and copies to dst (host or device).  *bytes receives the size; dst may be NULL to query. */
int coarse_halo_pack(cd_context *ctx, const cd_field *in, void *dst, int dst_on_device, size_t *bytes,
                     void *stream);

/* One halo exchange of `in` with the context's transport and nothing else (no stencil): the
 * pack (+ transfer), the exchange and the arrival wait, all ordered on `stream`; then the
 * received buffer (R13 wire order, *bytes long) is copied to dst (host or device;
 * NULL: no copy -- e.g. to time the exchange alone).  Collective like coarse_dslash_apply. */
int coarse_halo_exchange(cd_context *ctx, const cd_field *in, void *dst, int dst_on_device, size_t *bytes,
                         void *stream);

/* Write the L2-flush scratch (bench utility): a kernel writing `bytes` of device memory. */
int cd_flush_l2(cd_context *ctx, size_t bytes, void *stream);

/* ------------------------------------------------------------------ halo plan (host only) */

/* The domain decomposition and halo wire layout of one rank (R13), computed on the
 * host without touching a GPU; the library's own pack / exchange / halo-term path uses exactly
 * this plan.  Exchange schedule for every split dim mu: send block A to nbr_rank[mu][0] (+mu)
 * and block B to nbr_rank[mu][1] (-mu); receive block A from nbr_rank[mu][1] and block B from
 * nbr_rank[mu][0], into the same offsets of the receive buffer.  A +mu hop of a face site reads
 * block B, a -mu hop block A; record f of a block is the face site with the other three
 * coordinates lexicographic (lowest mu fastest). */
typedef struct {
    int32_t local_dims[4];
    int32_t grid_coords[4];
    int64_t local_volume;
    int32_t split_mask;          /* bit mu: dim mu exchanged (P_mu > 1, or forced by self_mask) */
    int32_t nbr_rank[4][2];      /* [mu][0] = rank at +mu, [mu][1] = rank at -mu (periodic)    */
    int64_t face_sites[4];       /* sites of one face of dim mu (= V / L_mu)                    */
    int64_t record_bytes;        /* wire payload bytes per site (fp32: 8N, fp16: 4N)            */
    int64_t scale_bytes;         /* wire scale bytes per site (fp32: 0, fp16: 4)                */
    int64_t block_offset[4][2];  /* byte offset of block A / B of dim mu (0 if not split)       */
    int64_t block_bytes[4];      /* bytes of one block of dim mu, zero-padded to 16             */
    int64_t total_bytes;         /* send (= receive) buffer size                                */
} cd_halo_plan;

/* Fill *out for `rank` of the process grid in geom (self_mask as CD_OPT_HALO_SELF_MASK).
 * CD_ERR_INVALID / CD_ERR_UNSUPPORTED as cd_context_create's geometry checks. */
int cd_halo_plan_create(const cd_geometry *geom, int nranks, int rank, cd_precision prec, int32_t self_mask,
                        cd_halo_plan *out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* COARSE_DSLASH_H */
