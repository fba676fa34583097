/*
 * tnrd_oracle.c -- CPU float64 restatement of the reference TNRD inference
 * path.  TEST INFRASTRUCTURE ONLY: this file is the checker for the CUDA
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The shipped library
 * (paper_1702_07482_b200/csrc) never links or calls it.
 *
 * Parity pin: outputs are checked against golden vectors produced by the
 * real reference (tests/golden/make_golden.py imports specklediff from
 * /root/reference) in tests/test_oracle.py.
 *
 * What it restates (reference = /root/reference/pkg/src/specklediff):
 *   oracle_conv2d        imageops.py:53-72   same-size TRUE convolution of a
 *                        half-sample-symmetric ("np.pad symmetric") padded
 *                        image; z[y,x] = sum_{p,q in [-r,r]} k[r+p,r+q] *
 *                        img[mir(y-p), mir(x-q)]  (tests/test_imageops.py:8-30)
 *   rbf influence        influence.py:40-45 + diffusion.py:177
 *                        phi(z) = sum_j w_j exp(-(z-mu_j)^2 / (2 gamma^2)),
 *                        evaluated over ALL centres, j ascending.
 *   oracle_prox_idiv     speckle.py:103-121  (u~ + sqrt(u~^2 + 8 a lam f^2))/(2a),
 *                        a = 1 + 2 lam, f floored at 1e-6.
 *   oracle_stage         diffusion.py:171-194 force = sum_i conv2d(phi_i(conv2d(u,k_i)),
 *                        rot180(k_i)) accumulated i-ascending; u~ = u - force;
 *                        u_next = prox(u~, f, lam).
 *   oracle_run_diffusion diffusion.py:219-242 u0 = max(f, 1e-6); T stages;
 *                        non-finite check after every stage.
 *   oracle_speckle_field speckle.py:51-61 amplitude speckle sqrt(G/L),
 *                        G ~ Gamma(L, 1), restated with the GPU path's
 *                        generator (Philox4x32-10, counter = pixel index /
 *                        block, Marsaglia-Tsang) in float64: the checker for
 *                        tnrd_sample_speckle.  The reference's numpy stream
 *                        (Generator(Philox).gamma) is matched in distribution
 *                        by the tests, not bitwise (no parallel equivalent).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_F_FLOOR 1e-6 /* speckle.py:21 */

/* ---- minimal pthread parallel-for over [0, n) (no OpenMP in this image) */
static int g_threads = 1;

typedef void (*range_fn)(long lo, long hi, void* ctx);
typedef struct { range_fn fn; void* ctx; long lo, hi; } par_job;

static void* par_worker(void* arg) {
    par_job* j = (par_job*)arg;
    j->fn(j->lo, j->hi, j->ctx);
    return NULL;
}

static void par_for(long n, range_fn fn, void* ctx) {
    int nt = g_threads;
    if (nt > n) nt = (int)n;
    if (nt <= 1) { fn(0, n, ctx); return; }
    pthread_t th[256];
    par_job jobs[256];
    if (nt > 256) nt = 256;
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx;
        jobs[t].lo = n * t / nt; jobs[t].hi = n * (t + 1) / nt;
    }
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, par_worker, &jobs[t]);
    par_worker(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

void oracle_set_threads(int n) {
    if (n <= 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        n = c > 0 ? (int)c : 1;
    }
    g_threads = n;
}

/* Half-sample symmetric reflection, repeated as np.pad(mode="symmetric")
 * does for pads wider than the image (imageops.py:65). */
static inline int mir(int j, int n) {
    if (n == 1) return 0;
    int period = 2 * n;
    j %= period;
    if (j < 0) j += period;
    return j < n ? j : period - 1 - j;
}

/* imageops.py:53-72 (conv2d): true convolution, mirror padded, same size. */
typedef struct { const double* img; int H, W; const double* k; int m; double* out; } conv_ctx;

static void conv_rows(long lo, long hi, void* vctx) {
    const conv_ctx* c = (const conv_ctx*)vctx;
    const double* img = c->img; const double* k = c->k; double* out = c->out;
    const int H = c->H, W = c->W, m = c->m, r = m / 2;
    for (int y = (int)lo; y < (int)hi; ++y) {
        for (int x = 0; x < W; ++x) {
            double s = 0.0;
            for (int p = -r; p <= r; ++p) {
                const double* row = img + (size_t)mir(y - p, H) * W;
                const double* krow = k + (size_t)(r + p) * m;
                for (int q = -r; q <= r; ++q)
                    s += krow[r + q] * row[mir(x - q, W)];
            }
            out[(size_t)y * W + x] = s;
        }
    }
}

static void conv_true_mirror(const double* img, int H, int W, const double* k,
                             int m, double* out) {
    conv_ctx c = {img, H, W, k, m, out};
    par_for(H, conv_rows, &c);
}

void oracle_conv2d(const double* img, int H, int W, const double* k, int m,
                   double* out) {
    conv_true_mirror(img, H, W, k, m, out);
}

/* speckle.py:111-121 */
void oracle_prox_idiv(const double* ut, const double* f, double lam,
                      double* out, long n) {
    const double a = 1.0 + 2.0 * lam;
    for (long i = 0; i < n; ++i) {
        double fi = f[i] > ORACLE_F_FLOOR ? f[i] : ORACLE_F_FLOOR;
        double root = sqrt(ut[i] * ut[i] + 8.0 * a * lam * fi * fi);
        out[i] = (ut[i] + root) / (2.0 * a);
    }
}

/* influence.py:40-45 and diffusion.py:177, all M centres */
typedef struct { const double* z; const double* w; const double* centers; int M; double c; double* phi; } rbf_ctx;

static void rbf_range(long lo, long hi, void* vctx) {
    const rbf_ctx* r = (const rbf_ctx*)vctx;
    for (long i = lo; i < hi; ++i) {
        double s = 0.0;
        for (int j = 0; j < r->M; ++j) {
            double d = r->z[i] - r->centers[j];
            s += r->w[j] * exp(d * d * r->c);
        }
        r->phi[i] = s;
    }
}

static void rbf_phi(const double* z, long n, const double* w,
                    const double* centers, int M, double gamma, double* phi) {
    rbf_ctx c = {z, w, centers, M, -0.5 / (gamma * gamma), phi};
    par_for(n, rbf_range, &c);
}

/* diffusion.py:171-181 (diffusion_force); kernels are the reference's k_i
 * (coeffs @ basis.T), nk*m*m row-major. */
void oracle_force(const double* u, int H, int W, int m, int nk, int M,
                  const double* kernels, const double* weights,
                  const double* centers, double gamma, double* force) {
    const size_t n = (size_t)H * W;
    double* z = (double*)malloc(n * sizeof(double));
    double* phi = (double*)malloc(n * sizeof(double));
    double* tmp = (double*)malloc(n * sizeof(double));
    double* krot = (double*)malloc((size_t)m * m * sizeof(double));
    memset(force, 0, n * sizeof(double));
    for (int i = 0; i < nk; ++i) {
        const double* k = kernels + (size_t)i * m * m;
        for (int t = 0; t < m * m; ++t) krot[t] = k[m * m - 1 - t]; /* imageops.py:48-50 */
        conv_true_mirror(u, H, W, k, m, z);
        rbf_phi(z, (long)n, weights + (size_t)i * M, centers, M, gamma, phi);
        conv_true_mirror(phi, H, W, krot, m, tmp);
        for (size_t p = 0; p < n; ++p) force[p] += tmp[p];
    }
    free(z); free(phi); free(tmp); free(krot);
}

/* diffusion.py:184-194 (diffusion_step, prox variant) */
void oracle_stage(const double* u, const double* f, int H, int W, int m,
                  int nk, int M, const double* kernels, const double* weights,
                  const double* centers, double gamma, double lam,
                  double* u_next) {
    const size_t n = (size_t)H * W;
    double* force = (double*)malloc(n * sizeof(double));
    oracle_force(u, H, W, m, nk, M, kernels, weights, centers, gamma, force);
    for (size_t p = 0; p < n; ++p) force[p] = u[p] - force[p];
    oracle_prox_idiv(force, f, lam, u_next, (long)n);
    free(force);
}

/* diffusion.py:149-156, 197-216 (projected comparison variant) */
void oracle_stage_projected(const double* u, const double* f, int H, int W, int m,
                            int nk, int M, const double* kernels, const double* weights,
                            const double* centers, double gamma, double lam,
                            double floor_, double* u_next) {
    const size_t n = (size_t)H * W;
    const double tau = 0.01 * floor_; /* PROJECTION_KNEE, diffusion.py:24 */
    oracle_force(u, H, W, m, nk, M, kernels, weights, centers, gamma, u_next);
    for (size_t p = 0; p < n; ++p) {
        const double ut = u[p] - u_next[p] - lam * (1.0 / u[p] - f[p] * f[p] / (u[p] * u[p] * u[p]));
        const double x = (ut - floor_) / tau;   /* logaddexp(0, x) */
        u_next[p] = floor_ + tau * ((x > 0 ? x : 0.0) + log1p(exp(-fabs(x))));
    }
}

int oracle_run_diffusion_ex(const double* f, int H, int W, int m, int nk, int T,
                            int M, const double* kernels, const double* weights,
                            const double* centers, double gamma,
                            const double* lam, int variant, double floor_,
                            double* u_out, int nthreads);

/* diffusion.py:219-242.  Returns -1 on success, else the first stage index
 * whose output is non-finite (the reference raises FloatingPointError). */
int oracle_run_diffusion(const double* f, int H, int W, int m, int nk, int T,
                         int M, const double* kernels, const double* weights,
                         const double* centers, double gamma,
                         const double* lam, double* u_out, int nthreads) {
    return oracle_run_diffusion_ex(f, H, W, m, nk, T, M, kernels, weights, centers,
                                   gamma, lam, 0, 1.0, u_out, nthreads);
}

int oracle_run_diffusion_ex(const double* f, int H, int W, int m, int nk, int T,
                            int M, const double* kernels, const double* weights,
                            const double* centers, double gamma,
                            const double* lam, int variant, double floor_,
                            double* u_out, int nthreads) {
    if (nthreads != 0) oracle_set_threads(nthreads);
    const size_t n = (size_t)H * W;
    double* u = (double*)malloc(n * sizeof(double));
    const double u0f = variant ? floor_ : ORACLE_F_FLOOR; /* diffusion.py:219-224 */
    for (size_t p = 0; p < n; ++p)
        u[p] = f[p] > u0f ? f[p] : u0f;
    int bad = -1;
    for (int t = 0; t < T; ++t) {
        if (variant)
            oracle_stage_projected(u, f, H, W, m, nk, M, kernels + (size_t)t * nk * m * m,
                                   weights + (size_t)t * nk * M, centers, gamma, lam[t],
                                   floor_, u_out);
        else
            oracle_stage(u, f, H, W, m, nk, M, kernels + (size_t)t * nk * m * m,
                         weights + (size_t)t * nk * M, centers, gamma, lam[t],
                         u_out);
        for (size_t p = 0; p < n; ++p) {
            if (!isfinite(u_out[p])) { bad = t; break; }
        }
        if (bad >= 0) break;
        memcpy(u, u_out, n * sizeof(double));
    }
    if (bad < 0) memcpy(u_out, u, n * sizeof(double));
    free(u);
    return bad;
}

int oracle_max_threads(void) { return g_threads; }

/* ---- speckle (see header) ------------------------------------------------ */

typedef struct { uint32_t v[4]; } ph4;

static ph4 philox10(ph4 c, uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.v[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.v[2];
        ph4 n;
        n.v[0] = (uint32_t)(p1 >> 32) ^ c.v[1] ^ k0;
        n.v[1] = (uint32_t)p1;
        n.v[2] = (uint32_t)(p0 >> 32) ^ c.v[3] ^ k1;
        n.v[3] = (uint32_t)p0;
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    ph4 c = {{ctr[0], ctr[1], ctr[2], ctr[3]}};
    c = philox10(c, key[0], key[1]);
    for (int i = 0; i < 4; ++i) out[i] = c.v[i];
}

static double u01d(uint32_t b) { return ((double)(b >> 8) + 0.5) / 16777216.0; }

static int mt_try_d(double d, double c, double x, double u, double* g) {
    const double t = 1.0 + c * x;
    if (t <= 0.0) return 0;
    const double v = t * t * t;
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) { *g = d * v; return 1; }
    return 0;
}

static void box_muller_d(uint32_t b1, uint32_t b2, double* n0, double* n1) {
    const double rad = sqrt(-2.0 * log(u01d(b1)));
    const double th = 2.0 * M_PI * u01d(b2) - M_PI;
    *n0 = -rad * cos(th);
    *n1 = -rad * sin(th);
}

/* sqrt(Gamma(L,1)/L) of the pixel at flat index idx (tnrd_speckle.cuh) */
static double speckle_px(uint64_t idx, int looks, uint32_t k0, uint32_t k1) {
    const double d = looks - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    for (uint32_t att = 0;; ++att) {
        ph4 in = {{(uint32_t)idx, (uint32_t)(idx >> 32), att, 0u}};
        const ph4 r = philox10(in, k0, k1);
        double n0, n1, g;
        box_muller_d(r.v[0], r.v[1], &n0, &n1);
        if (mt_try_d(d, c, n0, u01d(r.v[2]), &g)) return sqrt(g / looks);
        if (mt_try_d(d, c, n1, u01d(r.v[3]), &g)) return sqrt(g / looks);
    }
}

typedef struct { double* out; int looks, W; uint32_t k0, k1; uint64_t base; } sp_ctx;

static void speckle_range(long lo, long hi, void* vctx) {
    sp_ctx* c = (sp_ctx*)vctx;
    for (long i = lo; i < hi; ++i)
        c->out[i] = speckle_px(c->base + (uint64_t)i, c->looks, c->k0, c->k1);
}

/* field values of flat pixel indices [base, base + n), rows of width W */
void oracle_speckle_field(double* out, long n, int W, int looks, uint64_t seed, uint64_t base) {
    sp_ctx c = {out, looks, W, (uint32_t)seed, (uint32_t)(seed >> 32), base};
    par_for(n, speckle_range, &c);
}
