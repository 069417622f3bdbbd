/*
 * oracle/oracle.c -- float64 CPU oracle of the coarse-grid Dirac operator.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or link this code.  It shares no
 * code, header, table or helper with the CUDA library (paper_1612_07873_b200/csrc), and
 * the CUDA library never calls it.
 *
 * What it computes (§3.4 Eq. 3, read as DESIGN.md R1-R10):
 *
 *   y(x) = X(x) v(x) + sum_{mu=0..3} [ L_{2mu}(x) v(x+mu) + L_{2mu+1}(x) v(x-mu) ]
 *
 * on a periodic 4-D lattice, each L_k(x) a dense N x N complex matrix, N = 2*Nvec
 * (coarse spin 2 x Nvec colours).  Layouts:
 *   site  s = ((x3*L2 + x2)*L1 + x1)*L0 + x0         (Listing 2: x0 fastest)
 *   dof   i = sigma*Nvec + c                         (Listing 3: spin slower)
 *   hop   k = 2*mu + dir, dir 0 = +mu, dir 1 = -mu   (§6.3 "mu*2+dir"); k = 8: X
 *   links[((s*9 + k)*N + i)*N + j], v[s*N + i]       complex double, interleaved re/im
 *
 * Every function is the plain definition written out: no blocking, no fusion, fixed
 * term order (X first, then k = 0..7), OpenMP only over independent output sites
 * (the paper's own CPU path is "rudimentary OpenMP").
 *
 * Pins (tests/test_oracle_*.py): plane-wave closed form, unit impulse,
 * shift == numpy.roll, block-diagonal == numpy.matmul, identity, L=1 self hops,
 * tau3-hermiticity adjoint identity + negative control, <w,Dv> == <D^H w,v>,
 * dense assembly, partition emulation, face slicing == numpy slicing, fp16 quantiser
 * == numpy float16 cast.  No function here is "parity unpinned".
 */
#include <complex.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

typedef double complex cplx;

/* Thread count of the OpenMP loops (bench.py reports the oracle at 1 thread and at all cores). */
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int oracle_get_threads(void) { return omp_get_max_threads(); }

#define MAXN 128

/* ---------------------------------------------------------------- geometry */

/* PAPER.md:197 (§6.1, Listing 2): x[0] fastest, x[3] slowest. */
static int64_t site_of(const int L[4], const int x[4])
{
    return (((int64_t)x[3] * L[2] + x[2]) * L[1] + x[1]) * L[0] + x[0];
}

static void coords_of(const int L[4], int64_t s, int x[4])
{
    x[0] = (int)(s % L[0]); s /= L[0];
    x[1] = (int)(s % L[1]); s /= L[1];
    x[2] = (int)(s % L[2]); s /= L[2];
    x[3] = (int)s;
}

static int64_t volume_of(const int L[4])
{
    return (int64_t)L[0] * L[1] * L[2] * L[3];
}

/* Periodic neighbour x + step*mu_hat (R10: periodic in all four dims). */
static int64_t hop(const int L[4], const int x[4], int mu, int step)
{
    int y[4] = {x[0], x[1], x[2], x[3]};
    y[mu] = ((y[mu] + step) % L[mu] + L[mu]) % L[mu];
    return site_of(L, y);
}

/* Neighbour site index for each hop k = 0..8 of site s (k = 8: the site itself). */
void oracle_neighbours(const int L[4], int64_t s, int64_t out[9])
{
    int x[4];
    coords_of(L, s, x);
    for (int mu = 0; mu < 4; mu++) {
        out[2 * mu] = hop(L, x, mu, +1);
        out[2 * mu + 1] = hop(L, x, mu, -1);
    }
    out[8] = s;
}

/* ---------------------------------------------------------------- operator */

/* acc[i] += sum_j M[i][j] * u[j] */
static void matvec_acc(int N, const cplx *M, const cplx *u, cplx *acc)
{
    for (int i = 0; i < N; i++) {
        cplx a = 0;
        for (int j = 0; j < N; j++) a += M[(int64_t)i * N + j] * u[j];
        acc[i] += a;
    }
}

/* acc[i] += sum_j conj(M[j][i]) * u[j]    (M^H u) */
static void matvec_h_acc(int N, const cplx *M, const cplx *u, cplx *acc)
{
    for (int i = 0; i < N; i++) {
        cplx a = 0;
        for (int j = 0; j < N; j++) a += conj(M[(int64_t)j * N + i]) * u[j];
        acc[i] += a;
    }
}

/* One output site from its 9 link matrices and the 9 vectors they multiply
 * (links9[k], vn[k] = v(nbr_k(x)), k = 8 the diagonal).  Term order: X, then k = 0..7. */
void oracle_site_apply(int N, const double *links9, const double *vn, double *y)
{
    const cplx *Lk = (const cplx *)links9;
    const cplx *u = (const cplx *)vn;
    cplx acc[MAXN];
    for (int i = 0; i < N; i++) acc[i] = 0;
    matvec_acc(N, Lk + (int64_t)8 * N * N, u + (int64_t)8 * N, acc);
    for (int k = 0; k < 8; k++) matvec_acc(N, Lk + (int64_t)k * N * N, u + (int64_t)k * N, acc);
    memcpy(y, acc, sizeof(cplx) * N);
}

/* y = D v  (Eq. 3 as read in DESIGN.md R1-R3: all nine matrices stored at x, oriented). */
void oracle_apply(const int L[4], int N, const double *links_, const double *v_, double *y_)
{
    const cplx *links = (const cplx *)links_;
    const cplx *v = (const cplx *)v_;
    cplx *y = (cplx *)y_;
    const int64_t V = volume_of(L);
    const int64_t NN = (int64_t)N * N;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < V; s++) {
        int x[4];
        coords_of(L, s, x);
        cplx acc[MAXN];
        for (int i = 0; i < N; i++) acc[i] = 0;
        matvec_acc(N, links + (s * 9 + 8) * NN, v + s * N, acc);                  /* X(x) v(x)        */
        for (int mu = 0; mu < 4; mu++) {
            int64_t sf = hop(L, x, mu, +1), sb = hop(L, x, mu, -1);
            matvec_acc(N, links + (s * 9 + 2 * mu) * NN, v + sf * N, acc);         /* L_{2mu} v(x+mu)   */
            matvec_acc(N, links + (s * 9 + 2 * mu + 1) * NN, v + sb * N, acc);     /* L_{2mu+1} v(x-mu) */
        }
        for (int i = 0; i < N; i++) y[s * N + i] = acc[i];
    }
}

/* ---------------------------------------------------------------- matrix-free mode
 * y = D v exactly as oracle_apply, but every link matrix is regenerated from the test-input
 * recipe when it is needed instead of being read from an array, so the full-size configs
 * (M4 1.5 GB, M5 43.5 GB of fp64 links) can be checked on the whole
 * lattice with memory for the vectors only.  The generator is the
 * counter-based recipe of SURVEY §8(c) c.3 (splitmix64 over global indices), written out here
 * independently of synth/ (and of the CUDA library's generator); a pin checks this function
 * bit-for-bit against oracle_apply on synth.links() for every recipe.
 *   kind 0 general:   L_k(x) = G(x,k)
 *   kind 1 hermitian: L_{2mu}(x) = G(x,2mu); L_{2mu+1}(x)[i][j] = s_i s_j conj(G(x-mu,2mu)[j][i]);
 *                     X(x)[i][j] = (G(x,8)[i][j] + s_i s_j conj(G(x,8)[j][i])) / 2   (s = tau3 signs)
 *   kind 2 / 3: the same with gsite := 0 and tag 4 (translation invariant)
 * every entry then multiplied by 2^scale_log2 (exact). */
static uint64_t sm64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double u_of(uint64_t base, uint64_t ctr)
{
    const uint64_t h = sm64(base + ctr);
    return (double)((int64_t)(h >> 42) - ((int64_t)1 << 21)) * 0x1p-21;
}

/* G(gsite, k)[i][j], counter ((((gsite*9 + k)*N + i)*N + j)*2 + part) */
static void gen_G(uint64_t base, int64_t gsite, int k, int N, cplx *M)
{
    for (int i = 0; i < N; i++)
        for (int j = 0; j < N; j++) {
            const uint64_t c = (uint64_t)(((((gsite * 9 + k) * N + i) * N) + j) * 2);
            M[(int64_t)i * N + j] = u_of(base, c) + I * u_of(base, c + 1);
        }
}

/* the nine matrices of site x (global coordinates = local: the oracle holds the whole lattice) */
static void gen_site_links(const int L[4], int N, int kind, uint64_t base, double scale, const int x[4], cplx *L9,
                           cplx *tmp)
{
    const int ti = kind >= 2, herm = kind & 1;
    const int64_t NN = (int64_t)N * N;
    const int64_t gs = ti ? 0 : site_of(L, x);
    for (int k = 0; k < 9; k++) gen_G(base, gs, k, N, L9 + k * NN);
    if (herm) {
        const int nvec = N / 2;
        cplx *X = L9 + 8 * NN;
        memcpy(tmp, X, sizeof(cplx) * NN);
        for (int i = 0; i < N; i++)
            for (int j = 0; j < N; j++) {
                const double ss = ((i < nvec) == (j < nvec)) ? 1.0 : -1.0;
                X[(int64_t)i * N + j] = 0.5 * (tmp[(int64_t)i * N + j] + ss * conj(tmp[(int64_t)j * N + i]));
            }
        for (int mu = 0; mu < 4; mu++) {
            const int64_t gb = ti ? 0 : hop(L, x, mu, -1);
            gen_G(base, gb, 2 * mu, N, tmp);
            cplx *B = L9 + (2 * mu + 1) * NN;
            for (int i = 0; i < N; i++)
                for (int j = 0; j < N; j++) {
                    const double ss = ((i < nvec) == (j < nvec)) ? 1.0 : -1.0;
                    B[(int64_t)i * N + j] = ss * conj(tmp[(int64_t)j * N + i]);
                }
        }
    }
    if (scale != 1.0)
        for (int64_t e = 0; e < 9 * NN; e++) L9[e] *= scale;
}

int oracle_apply_generated(const int L[4], int N, int kind, uint64_t seed, int scale_log2, const double *v_,
                           double *y_)
{
    if (N > MAXN || kind < 0 || kind > 3) return -1;
    const cplx *v = (const cplx *)v_;
    cplx *y = (cplx *)y_;
    const int64_t V = volume_of(L);
    const int64_t NN = (int64_t)N * N;
    const uint64_t tag = kind >= 2 ? 4 : 1;
    const uint64_t base = sm64(seed ^ (tag << 56));
    const double scale = ldexp(1.0, scale_log2);
    int rc = 0;
#pragma omp parallel
    {
        cplx *L9 = malloc(sizeof(cplx) * 10 * NN);
        if (!L9) {
#pragma omp atomic write
            rc = -2;
        } else {
#pragma omp for schedule(dynamic, 16)
            for (int64_t s = 0; s < V; s++) {
                int x[4];
                coords_of(L, s, x);
                gen_site_links(L, N, kind, base, scale, x, L9, L9 + 9 * NN);
                cplx acc[MAXN];
                for (int i = 0; i < N; i++) acc[i] = 0;
                matvec_acc(N, L9 + 8 * NN, v + s * N, acc);                              /* X(x) v(x)        */
                for (int mu = 0; mu < 4; mu++) {
                    int64_t sf = hop(L, x, mu, +1), sb = hop(L, x, mu, -1);
                    matvec_acc(N, L9 + (2 * mu) * NN, v + sf * N, acc);                   /* L_{2mu} v(x+mu)   */
                    matvec_acc(N, L9 + (2 * mu + 1) * NN, v + sb * N, acc);               /* L_{2mu+1} v(x-mu) */
                }
                for (int i = 0; i < N; i++) y[s * N + i] = acc[i];
            }
            free(L9);
        }
    }
    return rc;
}

/* tau3 = diag(+1 x Nvec, -1 x Nvec) (PAPER.md:121 footnote 1; R5/R6). */
static void tau3(int64_t V, int N, const cplx *in, cplx *out)
{
    for (int64_t s = 0; s < V; s++)
        for (int i = 0; i < N; i++)
            out[s * N + i] = (i < N / 2) ? in[s * N + i] : -in[s * N + i];
}

/* y = tau3 D tau3 w: the library's "dagger" (R5).  Equal to D^H w iff the links
 * are tau3-hermitian (coarse gamma5-hermiticity, PAPER.md:121 footnote 1). */
void oracle_apply_dagger_tau3(const int L[4], int N, const double *links, const double *w_, double *y_)
{
    const int64_t V = volume_of(L);
    cplx *t = (cplx *)malloc(sizeof(cplx) * V * N);
    cplx *u = (cplx *)malloc(sizeof(cplx) * V * N);
    tau3(V, N, (const cplx *)w_, t);
    oracle_apply(L, N, links, (const double *)t, (double *)u);
    tau3(V, N, u, (cplx *)y_);
    free(t);
    free(u);
}

/* y = D^H w, the true adjoint, from its definition:
 *   (D^H w)(x) = X(x)^H w(x) + sum_mu [ L_{2mu}(x-mu)^H w(x-mu) + L_{2mu+1}(x+mu)^H w(x+mu) ]
 * (block (x', x) of D is L_{2mu}(x') when x = x'+mu and L_{2mu+1}(x') when x = x'-mu). */
void oracle_adjoint(const int L[4], int N, const double *links_, const double *w_, double *y_)
{
    const cplx *links = (const cplx *)links_;
    const cplx *w = (const cplx *)w_;
    cplx *y = (cplx *)y_;
    const int64_t V = volume_of(L);
    const int64_t NN = (int64_t)N * N;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < V; s++) {
        int x[4];
        coords_of(L, s, x);
        cplx acc[MAXN];
        for (int i = 0; i < N; i++) acc[i] = 0;
        matvec_h_acc(N, links + (s * 9 + 8) * NN, w + s * N, acc);
        for (int mu = 0; mu < 4; mu++) {
            int64_t sb = hop(L, x, mu, -1), sf = hop(L, x, mu, +1);
            matvec_h_acc(N, links + (sb * 9 + 2 * mu) * NN, w + sb * N, acc);
            matvec_h_acc(N, links + (sf * 9 + 2 * mu + 1) * NN, w + sf * N, acc);
        }
        for (int i = 0; i < N; i++) y[s * N + i] = acc[i];
    }
}

/* Dense D in C^{VN x VN} (row-major), assembled with += so that the L_mu = 1, 2 cases,
 * where several hops land on the same block, keep every term (R10). */
void oracle_dense(const int L[4], int N, const double *links_, double *D_)
{
    const cplx *links = (const cplx *)links_;
    cplx *D = (cplx *)D_;
    const int64_t V = volume_of(L);
    const int64_t NN = (int64_t)N * N, VN = V * N;
    memset(D, 0, sizeof(cplx) * VN * VN);
    for (int64_t s = 0; s < V; s++) {
        int64_t nb[9];
        oracle_neighbours(L, s, nb);
        for (int k = 0; k < 9; k++)
            for (int i = 0; i < N; i++)
                for (int j = 0; j < N; j++)
                    D[(s * N + i) * VN + nb[k] * N + j] += links[(s * 9 + k) * NN + (int64_t)i * N + j];
    }
}

/* ---------------------------------------------------------------- halo (multi-rank) */

/* Canonical face order (R13, "a single packing kernel ... for all
 * exchange dimensions"): for each split dim mu ascending: block A = the face sent to the
 * +mu neighbour (local x_mu = Lloc_mu - 1), then block B = the face sent to the -mu
 * neighbour (x_mu = 0).  Inside a face, sites are lexicographic over the other three
 * coordinates, lowest mu fastest.  Each block holds the site records (rec_bytes each)
 * followed, if scales != NULL, by that block's per-site scales (scale_bytes each); every
 * block is zero-padded to a multiple of 16 bytes (so 128-bit loads of any block are aligned).
 * Returns the number of bytes written (out may be NULL to query the size). */
size_t oracle_pack_halo(const int Lloc[4], const int split[4], const void *payload, size_t rec_bytes,
                        const void *scales, size_t scale_bytes, void *out)
{
    const unsigned char *p = (const unsigned char *)payload;
    const unsigned char *sc = (const unsigned char *)scales;
    unsigned char *o = (unsigned char *)out;
    size_t off = 0;
    for (int mu = 0; mu < 4; mu++) {
        if (!split[mu]) continue;
        int o3[3], n = 0;
        for (int nu = 0; nu < 4; nu++)
            if (nu != mu) o3[n++] = nu;
        int64_t F = (int64_t)Lloc[o3[0]] * Lloc[o3[1]] * Lloc[o3[2]];
        for (int blk = 0; blk < 2; blk++) {
            int xmu = (blk == 0) ? Lloc[mu] - 1 : 0;
            for (int pass = 0; pass < (sc ? 2 : 1); pass++) {
                size_t rb = pass == 0 ? rec_bytes : scale_bytes;
                const unsigned char *src = pass == 0 ? p : sc;
                for (int64_t f = 0; f < F; f++) {
                    int x[4];
                    int64_t t = f;
                    x[o3[0]] = (int)(t % Lloc[o3[0]]); t /= Lloc[o3[0]];
                    x[o3[1]] = (int)(t % Lloc[o3[1]]); t /= Lloc[o3[1]];
                    x[o3[2]] = (int)t;
                    x[mu] = xmu;
                    int64_t s = site_of(Lloc, x);
                    if (o) memcpy(o + off, src + (size_t)s * rb, rb);
                    off += rb;
                }
            }
            while (off % 16) {
                if (o) o[off] = 0;
                off++;
            }
        }
    }
    return off;
}

/* Emulate an apply distributed over a P[0] x P[1] x P[2] x P[3] process grid with explicit
 * halo buffers: every rank packs its faces (oracle_pack_halo), the blocks are delivered
 * (block A of rank r -> block A of rank r+mu, block B -> rank r-mu), and every rank applies
 * the stencil reading remote neighbours from its receive buffer.  Same term order as
 * oracle_apply, so the result must be bit-identical to it (pin P10).
 * Rank layout: lexicographic like sites, rank = ((c3*P2 + c2)*P1 + c1)*P0 + c0. */
void oracle_partitioned_apply(const int Lg[4], const int P[4], int N, const double *links_,
                              const double *v_, double *y_)
{
    const cplx *links = (const cplx *)links_;
    const cplx *v = (const cplx *)v_;
    cplx *y = (cplx *)y_;
    int Ll[4], split[4];
    for (int mu = 0; mu < 4; mu++) {
        Ll[mu] = Lg[mu] / P[mu];
        split[mu] = P[mu] > 1;
    }
    const int nranks = P[0] * P[1] * P[2] * P[3];
    const int64_t Vl = volume_of(Ll);
    const int64_t NN = (int64_t)N * N;
    const size_t rec = sizeof(cplx) * N;
    const size_t hbytes = oracle_pack_halo(Ll, split, NULL, rec, NULL, 0, NULL);
    cplx **vloc = (cplx **)calloc(nranks, sizeof(cplx *));
    unsigned char **send = (unsigned char **)calloc(nranks, sizeof(void *));
    unsigned char **recv = (unsigned char **)calloc(nranks, sizeof(void *));
    int (*rc)[4] = calloc(nranks, sizeof(*rc));
    /* scatter the global field into per-rank local fields, and pack */
    for (int r = 0; r < nranks; r++) {
        int t = r;
        for (int mu = 0; mu < 4; mu++) { rc[r][mu] = t % P[mu]; t /= P[mu]; }
        vloc[r] = (cplx *)malloc(rec * Vl);
        for (int64_t sl = 0; sl < Vl; sl++) {
            int xl[4], xg[4];
            coords_of(Ll, sl, xl);
            for (int mu = 0; mu < 4; mu++) xg[mu] = rc[r][mu] * Ll[mu] + xl[mu];
            memcpy(vloc[r] + sl * N, v + site_of(Lg, xg) * N, rec);
        }
        send[r] = (unsigned char *)malloc(hbytes ? hbytes : 1);
        recv[r] = (unsigned char *)malloc(hbytes ? hbytes : 1);
        oracle_pack_halo(Ll, split, vloc[r], rec, NULL, 0, send[r]);
    }
    /* deliver: block A (to +mu) lands in the +mu neighbour's block A, block B in the -mu one's */
    for (int r = 0; r < nranks; r++) {
        size_t off = 0;
        for (int mu = 0; mu < 4; mu++) {
            if (!split[mu]) continue;
            size_t fb = rec * (size_t)(Vl / Ll[mu]);
            for (int blk = 0; blk < 2; blk++) {
                int c[4] = {rc[r][0], rc[r][1], rc[r][2], rc[r][3]};
                c[mu] = (c[mu] + (blk == 0 ? 1 : -1) + P[mu]) % P[mu];
                int dst = ((c[3] * P[2] + c[2]) * P[1] + c[1]) * P[0] + c[0];
                memcpy(recv[dst] + off, send[r] + off, fb);
                off += fb;
            }
        }
    }
    /* local apply; remote neighbours are read from the receive buffer */
    for (int r = 0; r < nranks; r++) {
        for (int64_t sl = 0; sl < Vl; sl++) {
            int xl[4], xg[4];
            coords_of(Ll, sl, xl);
            for (int mu = 0; mu < 4; mu++) xg[mu] = rc[r][mu] * Ll[mu] + xl[mu];
            int64_t sg = site_of(Lg, xg);
            const cplx *nbv[9];
            for (int mu = 0; mu < 4; mu++) {
                for (int dir = 0; dir < 2; dir++) {
                    int step = dir == 0 ? +1 : -1;
                    int edge = dir == 0 ? (xl[mu] == Ll[mu] - 1) : (xl[mu] == 0);
                    if (split[mu] && edge) {
                        /* +mu hop reads block B (sent by the +mu neighbour), -mu hop block A */
                        size_t off = 0;
                        for (int nu = 0; nu < mu; nu++)
                            if (split[nu]) off += 2 * rec * (size_t)(Vl / Ll[nu]);
                        if (dir == 0) off += rec * (size_t)(Vl / Ll[mu]);
                        int o3[3], n = 0;
                        for (int nu = 0; nu < 4; nu++)
                            if (nu != mu) o3[n++] = nu;
                        int64_t f = ((int64_t)xl[o3[2]] * Ll[o3[1]] + xl[o3[1]]) * Ll[o3[0]] + xl[o3[0]];
                        nbv[2 * mu + dir] = (const cplx *)(recv[r] + off + (size_t)f * rec);
                    } else {
                        nbv[2 * mu + dir] = vloc[r] + hop(Ll, xl, mu, step) * N;
                    }
                }
            }
            nbv[8] = vloc[r] + sl * N;
            cplx acc[MAXN];
            for (int i = 0; i < N; i++) acc[i] = 0;
            matvec_acc(N, links + (sg * 9 + 8) * NN, nbv[8], acc);
            for (int k = 0; k < 8; k++) matvec_acc(N, links + (sg * 9 + k) * NN, nbv[k], acc);
            for (int i = 0; i < N; i++) y[sg * N + i] = acc[i];
        }
    }
    for (int r = 0; r < nranks; r++) {
        free(vloc[r]);
        free(send[r]);
        free(recv[r]);
    }
    free(vloc);
    free(send);
    free(recv);
    free(rc);
}

/* ---------------------------------------------------------------- 16-bit storage */

/* Half-precision storage ("custom 16-bit ... storage format" with a scale;
 * DESIGN.md R12): per record (a site's vector, or one (site, k) matrix):
 *   xf = fp32_rn(x);  s = max |xf|  (over all re and im parts);
 *   q  = fp16_rn(xf / s)   (correctly rounded fp32 division, then round-to-nearest-even);
 *   s == 0 -> every q = +0.
 * Both roundings are IEEE: C's double->float cast and _Float16 conversion (x86-64 SSE). */
void oracle_quantise_fp16(int64_t nrec, int64_t reals_per_rec, const double *x, uint16_t *q, float *scale)
{
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrec; r++) {
        const double *xr = x + r * reals_per_rec;
        float s = 0.0f;
        for (int64_t e = 0; e < reals_per_rec; e++) {
            float a = fabsf((float)xr[e]);
            if (a > s) s = a;
        }
        scale[r] = s;
        for (int64_t e = 0; e < reals_per_rec; e++) {
            _Float16 h = (s == 0.0f) ? (_Float16)0.0f : (_Float16)((float)xr[e] / s);
            uint16_t bits;
            memcpy(&bits, &h, 2);
            q[r * reals_per_rec + e] = bits;
        }
    }
}

/* x' = float(q) * s, returned in double (exact). */
void oracle_dequantise_fp16(int64_t nrec, int64_t reals_per_rec, const uint16_t *q, const float *scale,
                            double *x)
{
    for (int64_t r = 0; r < nrec; r++)
        for (int64_t e = 0; e < reals_per_rec; e++) {
            _Float16 h;
            memcpy(&h, q + r * reals_per_rec + e, 2);
            x[r * reals_per_rec + e] = (double)((float)h * scale[r]);
        }
}

/* ---------------------------------------------------------------- even-odd */

/* Inverse of an N x N complex matrix by Gauss-Jordan elimination with partial pivoting
 * (textbook; fp64).  Returns 0 on success, -1 if singular. */
int oracle_invert(int N, const double *A_, double *Ainv_)
{
    const cplx *A = (const cplx *)A_;
    cplx *Ainv = (cplx *)Ainv_;
    cplx *M = (cplx *)malloc(sizeof(cplx) * N * 2 * N);
    for (int i = 0; i < N; i++)
        for (int j = 0; j < 2 * N; j++)
            M[i * 2 * N + j] = j < N ? A[i * N + j] : (j - N == i ? 1.0 : 0.0);
    for (int c = 0; c < N; c++) {
        int p = c;
        for (int i = c + 1; i < N; i++)
            if (cabs(M[i * 2 * N + c]) > cabs(M[p * 2 * N + c])) p = i;
        if (cabs(M[p * 2 * N + c]) == 0.0) {
            free(M);
            return -1;
        }
        if (p != c)
            for (int j = 0; j < 2 * N; j++) {
                cplx t = M[c * 2 * N + j];
                M[c * 2 * N + j] = M[p * 2 * N + j];
                M[p * 2 * N + j] = t;
            }
        cplx piv = M[c * 2 * N + c];
        for (int j = 0; j < 2 * N; j++) M[c * 2 * N + j] /= piv;
        for (int i = 0; i < N; i++) {
            if (i == c) continue;
            cplx f = M[i * 2 * N + c];
            if (f == 0) continue;
            for (int j = 0; j < 2 * N; j++) M[i * 2 * N + j] -= f * M[c * 2 * N + j];
        }
    }
    for (int i = 0; i < N; i++)
        for (int j = 0; j < N; j++) Ainv[i * N + j] = M[i * 2 * N + N + j];
    free(M);
    return 0;
}

/* Even-odd Schur complement (red-black preconditioning, §3.3, used on all MG
 * levels), written from its definition on the full lattice:
 *     y_e = X_e v_e - D_eo X_o^{-1} D_oe v_e
 * where site parity = (x0+x1+x2+x3) mod 2 (every L_mu even), D_oe = the hopping terms from
 * even to odd sites, D_eo from odd to even.  v and y are FULL fields [V][N]; only their even
 * sites are read / written (odd sites of y are set to 0).  Returns -1 if an X_o is singular. */
int oracle_schur_apply(const int L[4], int N, const double *links_, const double *v_, double *y_)
{
    const cplx *links = (const cplx *)links_;
    const cplx *v = (const cplx *)v_;
    cplx *y = (cplx *)y_;
    const int64_t V = volume_of(L);
    const int64_t NN = (int64_t)N * N;
    cplx *t = (cplx *)calloc((size_t)V * N, sizeof(cplx));
    cplx *Xi = (cplx *)malloc(sizeof(cplx) * NN);
    int status = 0;
    for (int64_t s = 0; s < V && status == 0; s++) {   /* t_o = X_o^{-1} D_oe v_e */
        int x[4];
        coords_of(L, s, x);
        if (((x[0] + x[1] + x[2] + x[3]) & 1) == 0) continue;
        cplx u[MAXN];
        for (int i = 0; i < N; i++) u[i] = 0;
        int64_t nb[9];
        oracle_neighbours(L, s, nb);
        for (int k = 0; k < 8; k++) matvec_acc(N, links + (s * 9 + k) * NN, v + nb[k] * N, u);
        if (oracle_invert(N, (const double *)(links + (s * 9 + 8) * NN), (double *)Xi) != 0) {
            status = -1;
            break;
        }
        for (int i = 0; i < N; i++) {
            cplx a = 0;
            for (int j = 0; j < N; j++) a += Xi[i * N + j] * u[j];
            t[s * N + i] = a;
        }
    }
    for (int64_t s = 0; s < V; s++) {                  /* y_e = X_e v_e - D_eo t_o */
        int x[4];
        coords_of(L, s, x);
        cplx acc[MAXN];
        for (int i = 0; i < N; i++) acc[i] = 0;
        if (((x[0] + x[1] + x[2] + x[3]) & 1) == 0) {
            cplx hopsum[MAXN];
            for (int i = 0; i < N; i++) hopsum[i] = 0;
            int64_t nb[9];
            oracle_neighbours(L, s, nb);
            matvec_acc(N, links + (s * 9 + 8) * NN, v + s * N, acc);
            for (int k = 0; k < 8; k++) matvec_acc(N, links + (s * 9 + k) * NN, t + nb[k] * N, hopsum);
            for (int i = 0; i < N; i++) acc[i] -= hopsum[i];
        }
        for (int i = 0; i < N; i++) y[s * N + i] = acc[i];
    }
    free(t);
    free(Xi);
    return status;
}

/* ---------------------------------------------------------------- transfer operators
 *
 * Adaptive geometric aggregation (§3.4, setup steps 3-4; kernels §6.6):
 * the fine lattice Lf = Lc * B (regular non-overlapping hypercube aggregates of B0 x B1 x B2 x B3
 * fine sites, "regular non-overlapping hypercubes"); fine site xf belongs to the aggregate
 * (coarse site) xc = floor(xf / B).  A fine site carries Ns spins x Nc colours, dof r = s*Nc + a
 * (spin slower, as on the coarse grid).  Chirality-preserving aggregation (P:121 fn. 1): spins
 * s < Ns/2 form chirality 0, the rest chirality 1 (R20), so coarse dof i = sigma*Nvec + k.
 * Basis (the prolongator's columns): W[((sf*Ns + s)*Nc + a)*Nvec + k], complex.
 *
 *   prolong : vf(xf, s, a)      = sum_k W(xf, s, a, k) vc(xc(xf), chi(s)*Nvec + k)
 *   restrict: vc(xc, sigma*Nvec + k) = sum_{xf in xc} sum_{s: chi(s)=sigma} sum_a conj(W(xf,s,a,k)) vf(xf,s,a)
 *             (restrictor = P^dagger)
 */

static int64_t aggregate_of(const int Lc[4], const int B[4], const int xf[4])
{
    int xc[4] = {xf[0] / B[0], xf[1] / B[1], xf[2] / B[2], xf[3] / B[3]};
    return site_of(Lc, xc);
}

/* Prolongator: a gather per fine dof. */
void oracle_prolong(const int Lc[4], const int B[4], int Ns, int Nc, int Nvec, const double *W_, const double *vc_,
                    double *vf_)
{
    const cplx *W = (const cplx *)W_;
    const cplx *vc = (const cplx *)vc_;
    cplx *vf = (cplx *)vf_;
    const int Lf[4] = {Lc[0] * B[0], Lc[1] * B[1], Lc[2] * B[2], Lc[3] * B[3]};
    const int64_t Vf = volume_of(Lf);
    const int N = 2 * Nvec;
#pragma omp parallel for schedule(static)
    for (int64_t sf = 0; sf < Vf; sf++) {
        int xf[4];
        coords_of(Lf, sf, xf);
        const int64_t xc = aggregate_of(Lc, B, xf);
        for (int s = 0; s < Ns; s++) {
            const int chi = s < Ns / 2 ? 0 : 1;
            for (int a = 0; a < Nc; a++) {
                cplx acc = 0;
                for (int k = 0; k < Nvec; k++)
                    acc += W[((sf * Ns + s) * Nc + a) * Nvec + k] * vc[xc * N + chi * Nvec + k];
                vf[(sf * Ns + s) * Nc + a] = acc;
            }
        }
    }
}

/* Restrictor = P^dagger, written as its definition: for every coarse dof, the sum over
 * the aggregate's fine sites (fine site order), spins of that chirality and colours. */
void oracle_restrict(const int Lc[4], const int B[4], int Ns, int Nc, int Nvec, const double *W_, const double *vf_,
                     double *vc_)
{
    const cplx *W = (const cplx *)W_;
    const cplx *vf = (const cplx *)vf_;
    cplx *vc = (cplx *)vc_;
    const int Lf[4] = {Lc[0] * B[0], Lc[1] * B[1], Lc[2] * B[2], Lc[3] * B[3]};
    const int64_t Vf = volume_of(Lf), Vc = volume_of(Lc);
    const int N = 2 * Nvec;
    for (int64_t i = 0; i < Vc * N; i++) vc[i] = 0;
    for (int64_t sf = 0; sf < Vf; sf++) {
        int xf[4];
        coords_of(Lf, sf, xf);
        const int64_t xc = aggregate_of(Lc, B, xf);
        for (int s = 0; s < Ns; s++) {
            const int chi = s < Ns / 2 ? 0 : 1;
            for (int a = 0; a < Nc; a++)
                for (int k = 0; k < Nvec; k++)
                    vc[xc * N + chi * Nvec + k] +=
                        conj(W[((sf * Ns + s) * Nc + a) * Nvec + k]) * vf[(sf * Ns + s) * Nc + a];
        }
    }
}

/* Setup step 3: per aggregate and chirality, the block of basis rows (fine sites of the
 * aggregate in fine site order, spins of that chirality, colours) x Nvec columns is replaced by
 * the Q of its QR decomposition, computed by modified Gram-Schmidt in column order (R has a
 * positive real diagonal).  In place.  Returns -1 if a block is rank deficient: a column whose
 * norm after projection is <= 1e-10 x its norm before (R21). */
int oracle_block_orthonormalise(const int Lc[4], const int B[4], int Ns, int Nc, int Nvec, double *W_)
{
    cplx *W = (cplx *)W_;
    const int Lf[4] = {Lc[0] * B[0], Lc[1] * B[1], Lc[2] * B[2], Lc[3] * B[3]};
    const int64_t Vf = volume_of(Lf), Vc = volume_of(Lc);
    const int64_t Bvol = (int64_t)B[0] * B[1] * B[2] * B[3];
    const int64_t M = Bvol * (Ns / 2) * Nc;   /* rows of one (aggregate, chirality) block */
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * Vc * 2 * M);   /* row -> offset of W(.., k=0) */
    int64_t *fill = (int64_t *)calloc((size_t)Vc * 2, sizeof(int64_t));
    for (int64_t sf = 0; sf < Vf; sf++) {
        int xf[4];
        coords_of(Lf, sf, xf);
        const int64_t xc = aggregate_of(Lc, B, xf);
        for (int s = 0; s < Ns; s++) {
            const int chi = s < Ns / 2 ? 0 : 1;
            for (int a = 0; a < Nc; a++) {
                const int64_t blk = xc * 2 + chi;
                rows[blk * M + fill[blk]++] = ((sf * Ns + s) * Nc + a) * Nvec;
            }
        }
    }
    int status = 0;
    for (int64_t blk = 0; blk < Vc * 2 && status == 0; blk++) {
        const int64_t *r = rows + blk * M;
        for (int k = 0; k < Nvec; k++) {
            double nrm0 = 0;
            for (int64_t m = 0; m < M; m++) nrm0 += creal(W[r[m] + k]) * creal(W[r[m] + k]) +
                                                   cimag(W[r[m] + k]) * cimag(W[r[m] + k]);
            for (int j = 0; j < k; j++) {                 /* v_k -= <q_j, v_k> q_j */
                cplx d = 0;
                for (int64_t m = 0; m < M; m++) d += conj(W[r[m] + j]) * W[r[m] + k];
                for (int64_t m = 0; m < M; m++) W[r[m] + k] -= d * W[r[m] + j];
            }
            double nrm = 0;
            for (int64_t m = 0; m < M; m++) nrm += creal(W[r[m] + k]) * creal(W[r[m] + k]) +
                                                  cimag(W[r[m] + k]) * cimag(W[r[m] + k]);
            nrm = sqrt(nrm);
            if (!(nrm > 1e-10 * sqrt(nrm0))) {           /* DESIGN.md R21: numerically dependent */
                status = -1;
                break;
            }
            for (int64_t m = 0; m < M; m++) W[r[m] + k] /= nrm;
        }
    }
    free(rows);
    free(fill);
    return status;
}
