// tnrd_capi.cu -- C ABI (include/tnrd.h) over the fused sm_100a stage kernel.
//
// The Python drop-in (paper_1702_07482_b200) binds these symbols with ctypes;
// nothing here depends on torch.  Host-side parameter preparation follows
// the reference in float64 (kernels k_i = coeffs @ basis.T are computed by
// the caller exactly as diffusion.py:76-77 does; this file only casts them
// and builds the RBF tables), then everything is uploaded once per model.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tnrd.h"
#include "tnrd_stage.cuh"
#include "tnrd_stage_adj.cuh"
#include "tnrd_speckle.cuh"
#include "tnrd_train.cuh"
// The tensor-core and dataflow stage kernels measured slower than the
// CUDA-core kernels and are built only with
// -DTNRD_EXPERIMENTS (tools/build_experiments.sh); the shipped library
// reports TNRD_EUNSUPPORTED for their modes.
#ifdef TNRD_EXPERIMENTS
#include "tnrd_stage_tc.cuh"
#include "tnrd_stage_tc3.cuh"
#include "tnrd_stage_zf.cuh"
#include "tnrd_stage_fused.cuh"
#endif

using namespace tnrd;

constexpr int kNkPad = 16;   // filters are padded to a multiple of 16 (zero filters)

// ----------------------------------------------------------------- errors

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                              \
    do {                                                                            \
        cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess)                                                      \
            return fail(TNRD_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

extern "C" const char* tnrd_last_error(void) { return g_err.c_str(); }
extern "C" const char* tnrd_version(void) { return "tnrd-b200 0.1.0 sm_100a"; }
extern "C" uint64_t tnrd_launch_count(void) { return g_launches.load(); }
extern "C" uint32_t tnrd_build_features(void) {
#ifdef TNRD_EXPERIMENTS
    return TNRD_FEATURE_EXPERIMENTS;
#else
    return 0u;
#endif
}
extern "C" void tnrd_launch_count_reset(void) { g_launches.store(0); }
#ifdef TNRD_BOUNDS
// debug bounds mode (tnrd_stage.cuh TNRD_ASSERT): violations so far --
// out4 = {count, kind, value, limit of the first}; clears the counters
extern "C" __attribute__((visibility("default"))) int tnrd_bounds_failures(unsigned int* out4) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out4, g_bounds_fail, 4 * sizeof(unsigned int)));
    unsigned int z[4] = {0, 0, 0, 0};
    CUDA_TRY(cudaMemcpyToSymbol(g_bounds_fail, z, sizeof(z)));
    return TNRD_OK;
}
#endif
#ifdef TNRD_PHASE_TRACE
// tools/phase_trace.py: read (and clear) the tile kernel's per-phase clocks
extern "C" __attribute__((visibility("default"))) int tnrd_phase_trace(unsigned long long* out8) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out8, g_phase, 8 * sizeof(unsigned long long)));
    unsigned long long z[8] = {0};
    CUDA_TRY(cudaMemcpyToSymbol(g_phase, z, sizeof(z)));
    return TNRD_OK;
}
#endif

// ----------------------------------------------------------------- model

struct tnrd_model {
    int m = 0, nk = 0, nk_pad = 0, T = 0, M = 0;
    int device = 0;
    bool fast = false;   // polynomial RBF table (else direct all-centre sum)
    int kp = 0;          // floats per filter in taps
    int tab_stride = 0;  // floats per filter in tab
    double mu0 = 0, delta = 0, gamma = 0;
    double zlo = 0, h = 0;  // polynomial intervals: centre j at zlo + j h
    int ni = 0;             // number of intervals
    int nip = 0;            // intervals rounded to 8 (whole 8-interval table blocks)
    double fit_err = 0;     // max |p(z) - phi(z)| over all filters/stages
    double fit_err32 = 0;   // same with the fp32 coefficients
    double fit_scale = 0;   // max sum_j |w_ij|
    // cubic RBF table of the parameter-space-taps kernels (tnrd_stage.cuh
    // rbf_cubic_s): intervals of width h3 = min(delta, gamma) / kCubicSub,
    // one float4 (c0..c3) each
    double h3 = 0;
    int ni3 = 0, tab3_stride = 0;
    double fit_err3 = 0, fit_err3_32 = 0;
    float* d_tab3 = nullptr;  // T * nk_pad * tab3_stride
    std::vector<double> lam;
    int variant = 0;          // 0 prox, 1 projected (tnrd_model_set_variant)
    double floor = 1.0;       // projection floor
    float* d_taps = nullptr;  // T * nk_pad * kp
    std::vector<float> h_taps;  // host copy (parameter-space taps, TapBlock)
    float* d_tab = nullptr;   // T * nk_pad * tab_stride
    // tensor-core forward GEMM operand (m in {3,5,7}): per stage
    // [nk_pad/16 groups][m][ksteps][2 prec][2 kc][16][4]
    float* d_bop = nullptr;
    size_t bop_stage = 0;     // floats per stage
    // z-field forward operand (tnrd_stage_zf.cuh, m <= 7, nk_pad <= 128): per
    // stage [m][ksteps][3 pieces][2 kc][nk_pad][4] of kf = rot180(k)
    float* d_zop = nullptr;
    size_t zop_stage = 0;
    // split-kernel partial-force workspaces, one per stream (launches on one
    // stream are ordered, so a stream's workspace is never used by two
    // kernels at once); nothing in them outlives a stage
    struct SplitBuf { void* ptr = nullptr; size_t bytes = 0; std::vector<long> key; };
    mutable std::mutex ws_mu;
    // workspaces outgrown by a larger request: a CUDA graph captured
    // earlier may still reference them, so they are freed only with the
    // model (never while a captured launch could replay into them)
    mutable std::vector<void*> retired;
    mutable std::map<cudaStream_t, SplitBuf> ws;
    // fused dataflow workspaces (counters | stage args | claim sequence |
    // partials), one per stream, rebuilt when the grid geometry changes
    mutable std::map<cudaStream_t, SplitBuf> fws;
    // z-field planes (tnrd_stage_zf.cuh), one per stream
    mutable std::map<cudaStream_t, SplitBuf> zws;
    // tensor-core adjoint (tnrd_stage_adj.cuh, mode 12): the GEMM's B operand
    // (per stage [ks][2 prec][2 kc][NB][4], built on first use) and the phi
    // workspaces, one per stream
    mutable float* d_aop = nullptr;
    mutable size_t aop_stage = 0;
    mutable std::map<cudaStream_t, SplitBuf> aws;
    // batch fork (tnrd_despeckle): per caller stream, a second stream and
    // the fork / join events (DESIGN.md §7b item 5)
    struct ForkRes { cudaStream_t s2 = nullptr; cudaEvent_t fork = nullptr, join = nullptr; };
    mutable std::map<cudaStream_t, ForkRes> forks;
};

// 0 = auto (the faster kernel as measured on B200: currently
// the CUDA-core kernels), 1 = CUDA-core only, 2 = tensor-core required,
// 3 / 4 = CUDA-core tile kernel with small / large tiles forced (tests), 5 =
// the phase-locked tcgen05 kernel (tnrd_stage_tc.cuh, kept for comparison),
// 6 / 7 = CUDA-core split kernel with large / small tiles forced (one
// launch pair per stage), 9 = fused dataflow despeckle (tnrd_despeckle /
// plans: all stages in one launch; opt-in), 8 = z-field stage
// (tnrd_stage_zf.cuh: tcgen05 forward over the image + TMA-fed RBF/adjoint),
// 10 / 11 = cluster kernel (one launch per stage: a tile's filter groups on
// the CTAs of a thread-block cluster, partial forces summed through
// distributed shared memory) with large / small tiles forced
static std::atomic<int> g_kernel_mode{0};
// tnrd_set_param_taps; -1 = not set (TNRD_PARAM_TAPS=0|1 gives the initial value)
static std::atomic<int> g_param_taps{-1};

extern "C" int tnrd_set_param_taps(int on) {
    g_param_taps.store(on ? 1 : 0);
    return TNRD_OK;
}

extern "C" int tnrd_set_stage_kernel(int mode) {
    if (mode < 0 || mode > 12) return fail(TNRD_EINVAL, "stage kernel mode must be in 0..12");
    g_kernel_mode.store(mode);
    return TNRD_OK;
}

// CTAs per cluster of the cluster kernels: 0 = by grid size (cluster_size()),
// 2..8 forced (the summation order, and with it the bits, depends on it)
static std::atomic<int> g_cluster_size{0};
extern "C" int tnrd_set_cluster_size(int ctas) {
    if (ctas != 0 && (ctas < 2 || ctas > kMaxCluster))
        return fail(TNRD_EINVAL, "cluster size must be 0 (auto) or 2..%d", kMaxCluster);
    g_cluster_size.store(ctas);
    return TNRD_OK;
}

// round-to-nearest (ties away) to tf32, as cvt.rna.tf32.f32
[[maybe_unused]] static float tf32_rna_host(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b = (b + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &b, 4);
    return r;
}

// phi(z) of one filter, as the reference evaluates it (influence.py:40-45).
// Centres further than 10 gamma from z contribute < e^-50 |w_j| and are
// skipped (model creation would otherwise cost seconds for C5-sized models).
static double phi_exact(const double* w, int M, double mu0, double delta, double gamma, double z) {
    const double reach = 10.0 * gamma / delta;
    const double t = (z - mu0) / delta;
    const int jlo = std::max(0, (int)std::floor(t - reach));
    const int jhi = std::min(M - 1, (int)std::ceil(t + reach));
    double s = 0.0;
    for (int j = jlo; j <= jhi; ++j) {
        const double d = z - (mu0 + j * delta);
        s += w[j] * std::exp(-d * d / (2.0 * gamma * gamma));
    }
    return s;
}

// Degree-7 interpolant of phi on [zc - h/2, zc + h/2] at Chebyshev nodes,
// as monomial coefficients in x = (z - zc)/h, written to out[slot(d)].
// Returns the max abs interpolation error (float64 coefficients) over 41
// check points and, in *err32, the same with the fp32-rounded coefficients
// the kernel uses.
template <int N = kPolyN, int NCHECK = 41>
static double fit_interval(const double* w, int M, double mu0, double delta, double gamma,
                           double zc, double h, float* out, double* err32) {
    long double A[N][N + 1];
    for (int k = 0; k < N; ++k) {
        const long double x = 0.5L * std::cos(M_PI * (2 * k + 1) / (2.0 * N));
        long double xp = 1.0L;
        for (int d = 0; d < N; ++d) { A[k][d] = xp; xp *= x; }
        A[k][N] = phi_exact(w, M, mu0, delta, gamma, zc + (double)x * h);
    }
    for (int c = 0; c < N; ++c) {  // Gaussian elimination, partial pivoting
        int piv = c;
        for (int r = c + 1; r < N; ++r)
            if (std::fabs((double)A[r][c]) > std::fabs((double)A[piv][c])) piv = r;
        if (piv != c)
            for (int k = 0; k <= N; ++k) std::swap(A[c][k], A[piv][k]);
        for (int r = 0; r < N; ++r) {
            if (r == c) continue;
            const long double f = A[r][c] / A[c][c];
            for (int k = c; k <= N; ++k) A[r][k] -= f * A[c][k];
        }
    }
    double c[N];
    float c32[N];
    for (int d = 0; d < N; ++d) {
        c[d] = (double)(A[d][N] / A[d][d]);
        c32[d] = (float)c[d];
        // degree 7: c0..c3 | c4..c7 at +32 floats (rbf_lo_offset); cubic: c0..c3
        out[N == 8 ? (d >> 2) * 32 + (d & 3) : d] = c32[d];
    }
    double err = 0.0, e32 = 0.0;
    for (int k = 0; k < NCHECK; ++k) {
        const double x = -0.5 + k / (double)(NCHECK - 1);
        double acc = 0.0, acc32 = 0.0;
        for (int d = N - 1; d >= 0; --d) {
            acc = acc * x + c[d];
            acc32 = acc32 * x + (double)c32[d];
        }
        const double ref = phi_exact(w, M, mu0, delta, gamma, zc + x * h);
        err = std::max(err, std::fabs(acc - ref));
        e32 = std::max(e32, std::fabs(acc32 - ref));
    }
    *err32 = e32;
    return err;
}

static bool finite_all(const double* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) return false;
    return true;
}

extern "C" int tnrd_model_create(int m, int nk, int T, int M, const double* kernels,
                                 const double* weights, double mu0, double delta,
                                 double gamma, const double* lam, int device,
                                 tnrd_model** out) {
    if (!out) return fail(TNRD_EINVAL, "out is NULL");
    *out = nullptr;
    if (m < 1 || m % 2 != 1) return fail(TNRD_EINVAL, "filter size must be odd, got %d", m);
    if (m != 3 && m != 5 && m != 7 && m != 9)
        return fail(TNRD_EUNSUPPORTED, "fused stage kernel is built for m in {3,5,7,9}, got %d", m);
    if (nk < 1) return fail(TNRD_EINVAL, "need at least one filter");
    if (T < 1) return fail(TNRD_EINVAL, "model needs at least one stage");
    if (M < 2) return fail(TNRD_EINVAL, "need at least 2 RBF centers");
    if (!kernels || !weights || !lam) return fail(TNRD_EINVAL, "NULL parameter array");
    if (!(delta > 0) || !(gamma > 0) || !std::isfinite(mu0))
        return fail(TNRD_EINVAL, "invalid RBF grid (delta=%g gamma=%g)", delta, gamma);
    if (!finite_all(kernels, (size_t)T * nk * m * m) || !finite_all(weights, (size_t)T * nk * M))
        return fail(TNRD_EINVAL, "model parameters contain non-finite values");
    for (int t = 0; t < T; ++t)
        if (!(lam[t] > 0) || !std::isfinite(lam[t]))
            return fail(TNRD_EINVAL, "lambda must be positive, got %g", lam[t]);

    auto* md = new tnrd_model();
    md->m = m; md->nk = nk; md->T = T; md->M = M; md->device = device;
    md->nk_pad = round_up(nk, kNkPad);  // zero filters beyond nk
    md->mu0 = mu0; md->delta = delta; md->gamma = gamma;
    md->lam.assign(lam, lam + T);
    md->kp = round_up(m * m, 4);
    // piecewise-polynomial RBF: intervals of width h = min(delta, gamma)
    // (one Gaussian std or less, so degree 11 reaches ~1e-11 of sum|w|) over
    // [mu_0 - 7 gamma, mu_{M-1} + 7 gamma]; beyond that phi < 3e-11 sum|w|.
    md->h = std::min(delta, gamma) / kPolySub;
    md->zlo = mu0 - 7.0 * gamma;
    const double zhi = mu0 + (M - 1) * delta + 7.0 * gamma;
    md->ni = (int)std::ceil((zhi - md->zlo) / md->h) + 1;
    // interval 0 and interval ni + 1 are all-zero guards: z beyond the fitted
    // range (phi < 3e-11 sum|w| there) reads phi = 0 -- the reference's exp
    // underflows to exactly 0 far out, which matters once |w| is huge
    md->nip = round_up(md->ni + 2, 8);   // whole 8-interval blocks (rbf_lo_offset)
    md->fast = (size_t)md->nip * kPolyN * kF <= 16384;  // <= 64 KB per group buffer
    md->tab_stride = md->fast ? md->nip * kPolyN : round_up(M, 4);

    // cubic table (parameter-space-taps kernels): same range, h / 5
    md->h3 = std::min(delta, gamma) / kCubicSub;
    md->ni3 = (int)std::ceil((zhi - md->zlo) / md->h3) + 1;
    md->tab3_stride = md->fast ? round_up(md->ni3 + 2, 8) * 4 : 0;   // + the two zero guards
    if (md->tab3_stride > kMaxCubicStride) md->tab3_stride = 0;   // PT kernels off

    const size_t ntap = (size_t)T * md->nk_pad * md->kp;
    const size_t ntab = (size_t)T * md->nk_pad * md->tab_stride;
    const size_t ntab3 = (size_t)T * md->nk_pad * md->tab3_stride;
    std::vector<float> taps(ntap, 0.0f), tab(ntab, 0.0f), tab3(ntab3, 0.0f);
    for (int t = 0; t < T; ++t) {
        for (int i = 0; i < nk; ++i) {
            const double* k = kernels + ((size_t)t * nk + i) * m * m;
            float* dst = taps.data() + ((size_t)t * md->nk_pad + i) * md->kp;
            for (int j = 0; j < m * m; ++j) dst[j] = (float)k[j];
            const double* w = weights + ((size_t)t * nk + i) * M;
            float* tb = tab.data() + ((size_t)t * md->nk_pad + i) * md->tab_stride;
            if (md->fast) {
                double sw = 0.0;
                for (int j = 0; j < M; ++j) sw += std::fabs(w[j]);
                md->fit_scale = std::max(md->fit_scale, sw);
                for (int q = 0; q < md->ni; ++q) {
                    double e32 = 0.0;
                    md->fit_err = std::max(md->fit_err,
                                           fit_interval(w, M, mu0, delta, gamma,
                                                        md->zlo + q * md->h, md->h,
                                                        tb + rbf_lo_offset(q + 1), &e32));
                    md->fit_err32 = std::max(md->fit_err32, e32);
                }
            } else {
                for (int j = 0; j < M; ++j) tb[j] = (float)w[j];
            }
        }
    }
    if (md->tab3_stride) {
        // (stage, filter) fits on all host threads
        const int jobs = T * nk;
        const int nth = std::max(1, std::min<int>(jobs, (int)std::thread::hardware_concurrency()));
        std::vector<double> e3(nth, 0.0), e3_32(nth, 0.0);
        std::vector<std::thread> th;
        for (int id = 0; id < nth; ++id)
            th.emplace_back([&, id] {
                for (int job = id; job < jobs; job += nth) {
                    const int t = job / nk, i = job % nk;
                    const double* w = weights + ((size_t)t * nk + i) * M;
                    float* tb = tab3.data() + ((size_t)t * md->nk_pad + i) * md->tab3_stride;
                    for (int q = 0; q < md->ni3; ++q) {
                        double e32 = 0.0;
                        e3[id] = std::max(e3[id], fit_interval<4, 9>(w, M, mu0, delta, gamma,
                                                                    md->zlo + q * md->h3, md->h3,
                                                                    tb + 4 * (q + 1), &e32));
                        e3_32[id] = std::max(e3_32[id], e32);
                    }
                }
            });
        for (auto& x : th) x.join();
        for (int id = 0; id < nth; ++id) {
            md->fit_err3 = std::max(md->fit_err3, e3[id]);
            md->fit_err3_32 = std::max(md->fit_err3_32, e3_32[id]);
        }
    }
    std::vector<float> bop, zop;
#ifdef TNRD_EXPERIMENTS
    // forward GEMM operand for the tensor-core kernel (kf = rot180(k), split
    // into tf32 hi + lo, K-major), see tnrd_stage_tc.cuh
    {
        const int ks = (m + 7) / 8, G = md->nk_pad / tc::kG;
        const size_t bo = 2 * tc::kG * 4;                       // floats per (a, kk, prec)
        md->bop_stage = (size_t)G * m * ks * 2 * bo;
        bop.assign(md->bop_stage * T, 0.0f);
        for (int t = 0; t < T; ++t)
            for (int g = 0; g < G; ++g)
                for (int a = 0; a < m; ++a)
                    for (int kk = 0; kk < ks; ++kk)
                        for (int kc = 0; kc < 2; ++kc)
                            for (int n = 0; n < tc::kG; ++n)
                                for (int e = 0; e < 4; ++e) {
                                    const int f = g * tc::kG + n, b = 8 * kk + 4 * kc + e;
                                    float v = 0.0f;
                                    if (f < nk && b < m)
                                        v = (float)kernels[(((size_t)t * nk + f) * m + (m - 1 - a)) * m + (m - 1 - b)];
                                    const float hi = tf32_rna_host(v);
                                    const size_t base = (size_t)t * md->bop_stage +
                                                        ((((size_t)g * m + a) * ks + kk) * 2) * bo;
                                    bop[base + (kc * tc::kG + n) * 4 + e] = hi;
                                    bop[base + bo + (kc * tc::kG + n) * 4 + e] = tf32_rna_host(v - hi);
                                }
    }
    // z-field forward operand: kf = rot180(k) split into 3 tf32 pieces
    // (hi, mid, lo), K-major [kc][n][4] per (tap row a, K-step, piece)
    if (m <= 7 && md->nk_pad <= 128) {
        const int ks = (m + 7) / 8, np = md->nk_pad;
        const size_t bo = 2 * (size_t)np * 4;
        md->zop_stage = (size_t)m * ks * zf::kPieces * bo;
        zop.assign(md->zop_stage * T, 0.0f);
        for (int t = 0; t < T; ++t)
            for (int a = 0; a < m; ++a)
                for (int kk = 0; kk < ks; ++kk)
                    for (int kc = 0; kc < 2; ++kc)
                        for (int n = 0; n < np; ++n)
                            for (int e = 0; e < 4; ++e) {
                                const int b = 8 * kk + 4 * kc + e;
                                float v = 0.0f;
                                if (n < nk && b < m)
                                    v = (float)kernels[(((size_t)t * nk + n) * m + (m - 1 - a)) * m + (m - 1 - b)];
                                float r = v;
                                for (int pc = 0; pc < zf::kPieces; ++pc) {
                                    const float h = tf32_rna_host(r);
                                    r = r - h;
                                    zop[(size_t)t * md->zop_stage + ((size_t)(a * ks + kk) * zf::kPieces + pc) * bo +
                                        ((size_t)kc * np + n) * 4 + e] = h;
                                }
                            }
    }
#endif
    {
        DeviceGuard dg(device);
        if (!zop.empty()) {
            cudaError_t ez = cudaMalloc(&md->d_zop, zop.size() * sizeof(float));
            if (ez == cudaSuccess)
                ez = cudaMemcpy(md->d_zop, zop.data(), zop.size() * sizeof(float), cudaMemcpyHostToDevice);
            if (ez != cudaSuccess) {
                cudaFree(md->d_zop);
                delete md;
                return fail(TNRD_ECUDA, "z-field operand upload failed: %s", cudaGetErrorString(ez));
            }
        }
        if (!bop.empty()) {
            cudaError_t eb = cudaMalloc(&md->d_bop, bop.size() * sizeof(float));
            if (eb == cudaSuccess)
                eb = cudaMemcpy(md->d_bop, bop.data(), bop.size() * sizeof(float), cudaMemcpyHostToDevice);
            if (eb != cudaSuccess) {
                cudaFree(md->d_bop);
                cudaFree(md->d_zop);
                delete md;
                return fail(TNRD_ECUDA, "tensor-core operand upload failed: %s", cudaGetErrorString(eb));
            }
        }
        cudaError_t e1 = cudaMalloc(&md->d_taps, ntap * sizeof(float));
        cudaError_t e2 = cudaMalloc(&md->d_tab, ntab * sizeof(float));
        if (e1 != cudaSuccess || e2 != cudaSuccess) {
            cudaFree(md->d_taps); cudaFree(md->d_tab); cudaFree(md->d_tab3); cudaFree(md->d_bop); cudaFree(md->d_zop);
            delete md;
            return fail(TNRD_ECUDA, "cudaMalloc of model parameters failed: %s",
                        cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
        }
        md->h_taps.assign(taps.begin(), taps.begin() + ntap);
        if (ntab3) {
            cudaError_t e5 = cudaMalloc(&md->d_tab3, ntab3 * sizeof(float));
            if (e5 == cudaSuccess)
                e5 = cudaMemcpy(md->d_tab3, tab3.data(), ntab3 * sizeof(float), cudaMemcpyHostToDevice);
            if (e5 != cudaSuccess) {
                cudaFree(md->d_taps); cudaFree(md->d_tab); cudaFree(md->d_tab3); cudaFree(md->d_bop);
                cudaFree(md->d_zop);
                delete md;
                return fail(TNRD_ECUDA, "cubic RBF table upload failed: %s", cudaGetErrorString(e5));
            }
        }
        cudaError_t e3 = cudaMemcpy(md->d_taps, taps.data(), ntap * sizeof(float), cudaMemcpyHostToDevice);
        cudaError_t e4 = cudaMemcpy(md->d_tab, tab.data(), ntab * sizeof(float), cudaMemcpyHostToDevice);
        if (e3 != cudaSuccess || e4 != cudaSuccess) {
            cudaFree(md->d_taps); cudaFree(md->d_tab); cudaFree(md->d_tab3); cudaFree(md->d_bop); cudaFree(md->d_zop);
            delete md;
            return fail(TNRD_ECUDA, "parameter upload failed: %s",
                        cudaGetErrorString(e3 != cudaSuccess ? e3 : e4));
        }
    }
    *out = md;
    return TNRD_OK;
}

extern "C" int tnrd_model_destroy(tnrd_model* md) {
    if (!md) return TNRD_OK;
    {
        DeviceGuard dg(md->device);
        cudaFree(md->d_taps);
        cudaFree(md->d_tab);
        cudaFree(md->d_tab3);
        cudaFree(md->d_bop);
        cudaFree(md->d_zop);
        cudaDeviceSynchronize();   // retired workspaces may back queued graph replays
        for (void* q : md->retired) cudaFree(q);
        for (auto& kv : md->ws) cudaFree(kv.second.ptr);
        for (auto& kv : md->zws) cudaFree(kv.second.ptr);
        for (auto& kv : md->aws) cudaFree(kv.second.ptr);
        cudaFree(md->d_aop);
        for (auto& kv : md->fws) cudaFree(kv.second.ptr);
        for (auto& kv : md->forks) {
            cudaStreamSynchronize(kv.second.s2);
            cudaStreamDestroy(kv.second.s2);
            cudaEventDestroy(kv.second.fork);
            cudaEventDestroy(kv.second.join);
        }
    }
    delete md;
    return TNRD_OK;
}

extern "C" int tnrd_model_rbf_fit(const tnrd_model* md, double* max_abs_err,
                                  double* max_abs_err_fp32, double* max_sum_abs_w,
                                  int* intervals) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (max_abs_err) *max_abs_err = md->fit_err;
    if (max_abs_err_fp32) *max_abs_err_fp32 = md->fit_err32;
    if (max_sum_abs_w) *max_sum_abs_w = md->fit_scale;
    if (intervals) *intervals = md->fast ? md->ni : 0;
    return TNRD_OK;
}

extern "C" int tnrd_model_rbf_fit_cubic(const tnrd_model* md, double* max_abs_err,
                                        double* max_abs_err_fp32, int* intervals) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (max_abs_err) *max_abs_err = md->fit_err3;
    if (max_abs_err_fp32) *max_abs_err_fp32 = md->fit_err3_32;
    if (intervals) *intervals = md->tab3_stride ? md->ni3 : 0;
    return TNRD_OK;
}

extern "C" int tnrd_model_set_variant(tnrd_model* md, int variant, double floor) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (variant != TNRD_VARIANT_PROX && variant != TNRD_VARIANT_PROJECTED)
        return fail(TNRD_EINVAL, "unknown variant %d", variant);
    if (variant == TNRD_VARIANT_PROJECTED && !(floor > 0) )
        return fail(TNRD_EINVAL, "projection floor must be positive");
    md->variant = variant;
    md->floor = floor;
    return TNRD_OK;
}

extern "C" int tnrd_model_info(const tnrd_model* md, int* m, int* nk, int* T, int* M, int* fast) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (m) *m = md->m;
    if (nk) *nk = md->nk;
    if (T) *T = md->T;
    if (M) *M = md->M;
    if (fast) *fast = md->fast ? 1 : 0;
    return TNRD_OK;
}

// ----------------------------------------------------------------- status

extern "C" int tnrd_status_reset(uint32_t* d_status, void* stream) {
    if (!d_status) return fail(TNRD_EINVAL, "status is NULL");
    CUDA_TRY(cudaMemsetAsync(d_status, 0xFF, TNRD_STATUS_WORDS * sizeof(uint32_t),
                             (cudaStream_t)stream));
    return TNRD_OK;
}

extern "C" int tnrd_status_decode(const uint32_t* h, int* bad_stage) {
    if (bad_stage) *bad_stage = -1;
    const uint32_t fflags = ~h[1];
    if (fflags & TNRD_STATUS_F_NONFINITE) return fail(TNRD_EINVAL, "f contains non-finite values");
    if (fflags & TNRD_STATUS_F_NEGATIVE) return fail(TNRD_EINVAL, "observation must be nonnegative");
    if (h[0] != 0xFFFFFFFFu) {
        if (bad_stage) *bad_stage = (int)h[0];
        return fail(TNRD_ENONFINITE, "non-finite image after stage %d", (int)h[0]);
    }
    return TNRD_OK;
}

// ----------------------------------------------------------------- stage launch

// CUDA-core stage kernel configurations (tile, rows per forward block,
// rows per backward block, threads, filters per group, min CTAs/SM), chosen
// from the sweeps in DESIGN.md §5: small tiles keep a single 512^2 image
// spread over all 148 SMs; large tiles cut the phi-halo recompute
// (inflation 1.48 -> 1.23) once the grid has enough tiles.
// parameter-space taps kernels (stage_kernel_pt / stage_kernel_split_pt):
// forward blocking and CTAs per SM (the taps no longer hold registers)
#ifndef TNRD_PT_RF
#define TNRD_PT_RF 5
#endif
#ifndef TNRD_PT_SPLIT_RF
#define TNRD_PT_SPLIT_RF TNRD_PT_RF
#endif
#ifndef TNRD_PT_M9_RF
#define TNRD_PT_M9_RF 2
#endif
#ifndef TNRD_PT_MINB
#define TNRD_PT_MINB 2
#endif
// tile kernel with parameter-space taps: filters per group and CTAs per SM
// (the split kernel keeps SplitTile's groups: they size its workspace)
#ifndef TNRD_PT_TILE_F
#define TNRD_PT_TILE_F 2
#endif
#ifndef TNRD_PT_SPLIT_F
#define TNRD_PT_SPLIT_F 2
#endif
#ifndef TNRD_TILE_TM
#define TNRD_TILE_TM 2
#endif
#ifndef TNRD_SPLIT_TM
#define TNRD_SPLIT_TM 0
#endif
#ifndef TNRD_TILE_TM_M9
#define TNRD_TILE_TM_M9 3
#endif
#ifndef TNRD_SPLIT_TM_M9
#define TNRD_SPLIT_TM_M9 0
#endif
#ifndef TNRD_PT_TILE_MINB
#define TNRD_PT_TILE_MINB 2
#endif
// cluster kernel (one launch per stage on small grids): tap layout modes
#ifndef TNRD_CLUSTER_TM
#define TNRD_CLUSTER_TM 2
#endif
#ifndef TNRD_CLUSTER_TM_M9
#define TNRD_CLUSTER_TM_M9 3
#endif
static bool param_taps_enabled() {
    int v = g_param_taps.load();
    if (v < 0) {
        const char* e = std::getenv("TNRD_PARAM_TAPS");
        v = (e && e[0] == '0') ? 0 : 1;
        int expect = -1;
        g_param_taps.compare_exchange_strong(expect, v);
        v = g_param_taps.load();
    }
    return v != 0;
}

struct SmallTile { static constexpr int TH = 32, TW = 32, RF = 2, RB = 2, NT = 256, F = 4; };
#ifndef TNRD_LARGE_RF
#define TNRD_LARGE_RF 5
#endif
#ifndef TNRD_LARGE_MINB
#define TNRD_LARGE_MINB 2
#endif
#ifndef TNRD_LARGE_F
#define TNRD_LARGE_F 2
#endif
struct LargeTile { static constexpr int TH = 64, TW = 64, RF = TNRD_LARGE_RF, RB = 4, NT = 256, F = TNRD_LARGE_F; };
#ifndef TNRD_SPLIT_F
#define TNRD_SPLIT_F 2
#endif
// split kernel units: one filter per unit halves the granularity of the SM
// balance (a 512^2 image = 64 tiles x 48 units over 148 SMs)
#ifndef TNRD_SPLIT_TH
#define TNRD_SPLIT_TH 64
#endif
#ifndef TNRD_SPLIT_RB
#define TNRD_SPLIT_RB 4
#endif
struct SplitTile {
    static constexpr int TH = TNRD_SPLIT_TH, TW = 64, RF = TNRD_LARGE_RF, RB = TNRD_SPLIT_RB, NT = 256,
                         F = TNRD_SPLIT_F;
};


constexpr size_t kMaxSplitBytes = size_t(1) << 30;
// split workspace: the range-claim control words (fixed place: they must
// stay zeroed whatever partial sizes later launches write), then the partial
// forces
constexpr size_t kSplitCtlBytes = (kSplitCtlWords * sizeof(uint32_t) + 255) / 256 * 256;
static size_t split_alloc_bytes(size_t part_bytes) { return kSplitCtlBytes + part_bytes; }
// SM-aware split ranges (tnrd_stage.cuh SplitWs): measured on B200 slower
// than blockIdx ranges although it removes the 12-unit SMs (C2 636 ->
// 606 / 595 MPix/s with the heavy ranges on the first / last CTA of an SM,
// profiles/r02_split_map), so off by default
#ifndef TNRD_SPLIT_MAP
#define TNRD_SPLIT_MAP 0
#endif
constexpr bool kMapSplit = TNRD_SPLIT_MAP != 0;
static int sm_count();

#ifdef TNRD_EXPERIMENTS
// ---- fused dataflow despeckle (tnrd_stage_fused.cuh) ----------------------

constexpr int kMaxFusedStages = 8;

struct FusedSetup {
    StageArgs st[kMaxFusedStages];
    StageArgs* dst;
    int T;
};

// stage arguments -> device memory inside the launch sequence (graph-safe:
// no host buffer has to outlive the call)
__global__ void fused_setup_kernel(const FusedSetup s) {
    if ((int)threadIdx.x < s.T) s.dst[threadIdx.x] = s.st[threadIdx.x];
}

struct FusedLayout {
    size_t ctl, stargs, seq, part0, part1, bytes;
    int nclaims;
};

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// claim sequence: (stage, tile, group pair) ordered by tile + D * stage, with
// D = one tile row + 1 (the dependency reach) + one wave of claims
#ifndef TNRD_FUSED_CLAIM
#define TNRD_FUSED_CLAIM 2
#endif
constexpr int kFusedClaim = TNRD_FUSED_CLAIM;   // filter groups per claim

static std::vector<int> fused_sequence(int T, int tiles, int tiles_x, int ng, int grid) {
    const int pairs = (ng + kFusedClaim - 1) / kFusedClaim;
    const int lag = (grid + pairs - 1) / pairs;
    const int D = tiles_x + 1 + lag;
    std::vector<int> seq;
    seq.reserve((size_t)T * tiles * pairs);
    for (long w = 0; w < (long)D * (T - 1) + tiles; ++w)
        for (int t = 0; t < T; ++t) {
            const long tile = w - (long)D * t;
            if (tile < 0 || tile >= tiles) continue;
            for (int pr = 0; pr < pairs; ++pr) seq.push_back((t << 24) | ((int)tile << 6) | (kFusedClaim * pr));
        }
    return seq;
}

static FusedLayout fused_layout(int T, int tiles, int ng, int tpx, int nclaims) {
    FusedLayout L;
    L.ctl = 0;
    L.stargs = align256(sizeof(uint32_t) * (2 + 2 * (size_t)T * tiles));
    L.seq = L.stargs + align256(sizeof(StageArgs) * T);
    L.part0 = L.seq + align256(sizeof(int) * (size_t)nclaims);
    const size_t part = align256(sizeof(float) * (size_t)tiles * ng * tpx);
    L.part1 = L.part0 + part;
    L.bytes = L.part1 + part;
    L.nclaims = nclaims;
    return L;
}

// the stream's fused workspace for this geometry: (re)built outside capture
static int fused_workspace(const tnrd_model* md, cudaStream_t s, const std::vector<long>& key,
                           int T, int tiles, int tiles_x, int ng, int tpx, int grid, void** out,
                           FusedLayout* lay) {
    std::lock_guard<std::mutex> lk(md->ws_mu);
    auto& b = md->fws[s];
    if (b.key != key) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(s, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            return fail(TNRD_ECUDA, "fused workspace must be built before stream capture");
        const std::vector<int> seq = fused_sequence(T, tiles, tiles_x, ng, grid);
        const FusedLayout L = fused_layout(T, tiles, ng, tpx, (int)seq.size());
        if (b.ptr) md->retired.push_back(b.ptr);   // a captured graph may still use it
        b.ptr = nullptr;
        b.bytes = 0;
        b.key.clear();
        CUDA_TRY(cudaMalloc(&b.ptr, L.bytes));
        CUDA_TRY(cudaMemset(b.ptr, 0, L.stargs));   // cursor, counters, flags
        CUDA_TRY(cudaMemcpy(static_cast<char*>(b.ptr) + L.seq, seq.data(), seq.size() * sizeof(int),
                            cudaMemcpyHostToDevice));
        b.bytes = L.bytes;
        b.key = key;
    }
    const int pairs = (ng + kFusedClaim - 1) / kFusedClaim;
    *lay = fused_layout(T, tiles, ng, tpx, T * tiles * pairs);
    *out = b.ptr;
    return TNRD_OK;
}



#endif  // TNRD_EXPERIMENTS

// Launch with programmatic stream serialization: the kernel may be scheduled
// while its predecessor on the stream drains, and waits for it with
// griddepcontrol.wait before touching the predecessor's output (the split
// kernel's unit / reduction pair, and consecutive stages, overlap their
// launch latency this way).
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, int block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Same, as thread-block clusters of `cl` CTAs along x (stage_kernel_cl*).
template <class... KArgs, class... Args>
static cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, int block, size_t smem, int cl,
                                      cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)cl;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int MS, bool FAST, class T>
struct StageKernel {
    static constexpr int TH = T::TH, TW = T::TW, RB = T::RB, NT = T::NT, F = T::F;
    // m = 9 keeps 81 taps in registers: deeper forward blocking would spill
#ifndef TNRD_M9_RF
#define TNRD_M9_RF 2
#endif
    static constexpr int RF = MS >= 9 ? TNRD_M9_RF : T::RF;
    // 3 CTAs/SM fit the register file for m <= 7; m = 9 keeps 81 taps live
    static constexpr int MINB = T::TH == 64 ? TNRD_LARGE_MINB : (MS >= 9 ? 2 : 3);
    using C = StageCfg<MS, TH, TW, RF, RB, NT, F>;

    template <class K>
    static int prepare(K kern, int dev, uint64_t& attr_set, std::mutex& mu) {
        std::lock_guard<std::mutex> lk(mu);
        if (!(attr_set & (1ull << (dev & 63)))) {
            CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          160 * 1024));
            attr_set |= 1ull << (dev & 63);
        }
        return TNRD_OK;
    }

    // parameter-space taps (TapBlock, tnrd_stage.cuh): large tiles only (one
    // thread per output block, so the tap address is warp-uniform)
    // one thread per output block (no filter split: warp-uniform filter)
    static constexpr bool kPT = (T::TW / 4) * (T::TH / T::RB) == T::NT && FAST;
    // tap layout / FFMA2 mode per kernel (tnrd_stage.cuh TapLayout), as
    // measured on B200 (profiles/r02_ffma2): tile kernel TNRD_TILE_TM
    // (default 2: filter-pair forward + row-pair backward; C3 +7.7% over the
    // scalar kernel, 1 = row pairs only +4.4%), m = 9 TNRD_TILE_TM_M9 (default
    // 3: filter-pair forward, scalar backward on the same taps: C5 +7.9%);
    // split kernel TNRD_SPLIT_TM (default 0: scalar; 1 / 2 / 3 measured
    // C2 -2.5% / +-0 / -1.5%).  All modes give the scalar kernel's bits.
    static constexpr int kTmTile = PairTaps<MS>::kOn ? TNRD_TILE_TM : TNRD_TILE_TM_M9;
    static constexpr int kTmSplit = PairTaps<MS>::kOn ? TNRD_SPLIT_TM : TNRD_SPLIT_TM_M9;
    // cluster kernel (the tile kernel body, groups split over a cluster)
    static constexpr int kTmCluster = PairTaps<MS>::kOn ? TNRD_CLUSTER_TM : TNRD_CLUSTER_TM_M9;
    using TB = TapBlock<kMaxParamTaps>;
    // forward blocking (measured on B200): m = 7 RF = 5 (252 blocks per
    // filter for 256 threads); m = 9 RF = 2 (C5 172.5 MPix/s; RF = 3 167.4,
    // RF = 6 144.4, RF = 4 138)
    static constexpr int RF_PT = MS >= 9 ? TNRD_PT_M9_RF : TNRD_PT_RF;
    static constexpr int F_TILE_PT = TNRD_PT_TILE_F;
    using CPT = StageCfg<MS, TH, TW, RF_PT, RB, NT, F_TILE_PT>;
    static constexpr int F_SPLIT_PT = TNRD_PT_SPLIT_F;
    static constexpr int RF_SPLIT_PT = MS >= 9 ? TNRD_PT_M9_RF : TNRD_PT_SPLIT_RF;
    using CPS = StageCfg<MS, TH, TW, RF_SPLIT_PT, RB, NT, F_SPLIT_PT>;
    // filters per split unit (the parameter-space kernel has its own)
    static int split_f(const StageArgs& a) { return pt_fits(a) ? F_SPLIT_PT : F; }
    // htaps: this stage's taps on the host, [nk_pad][kp]
    static bool pt_fits(const StageArgs& a) {
        return kPT && param_taps_enabled() && a.tab3 != nullptr &&
               tap_floats<kTmTile, F_TILE_PT>(a.nk) <= sizeof(TB) / sizeof(float) &&
               tap_floats<kTmSplit, F_SPLIT_PT>(a.nk) <= sizeof(TB) / sizeof(float) &&
               tap_floats<kTmCluster, F_TILE_PT>(a.nk) <= sizeof(TB) / sizeof(float);
    }
    // shared memory of the PT kernels: u | phi[f] | one cubic table for f filters
    template <class CC, int FF>
    static size_t pt_smem(const StageArgs& a) {
        return sizeof(float) * ((size_t)CC::SU + (size_t)FF * CC::SPHI + (size_t)FF * a.tab3_stride);
    }
    // floats of the TapBlock for nk filters in groups of FF (zero filters pad
    // the last group)
    template <int TM, int FF>
    static size_t tap_floats(int nk) {
        return (size_t)((nk + FF - 1) / FF) * TapLayout<MS, C::KP, FF, TM>::group;
    }
    // htaps: [nk_pad][KP] row-major k (zero rows past nk) -> layout TM
    template <int TM, int FF>
    static void fill_taps(TB& tb, const float* htaps, int nk) {
        using TL = TapLayout<MS, C::KP, FF, TM>;
        const int ng = (nk + FF - 1) / FF;
        std::memset(tb.k, 0, sizeof(float) * tap_floats<TM, FF>(nk));
        for (int g = 0; g < ng; ++g) {
            float* grp = tb.k + (size_t)g * TL::group;
            for (int fi = 0; fi < FF; ++fi) {
                const float* k = htaps + (size_t)(g * FF + fi) * C::KP;   // nk_pad rows: in range
                float* bw = grp + TL::bwd0 + fi * TL::per_filter;
                if constexpr (TM == 0) {
                    std::memcpy(bw, k, sizeof(float) * C::KP);
                } else if constexpr (TM != 3) {
                    for (int A = 1; A < MS; ++A)   // row pairs Q[A][B] = (k[A][B], k[A-1][B])
                        for (int B = 0; B < MS; ++B) {
                            bw[2 * ((A - 1) * MS + B)] = k[A * MS + B];
                            bw[2 * ((A - 1) * MS + B) + 1] = k[(A - 1) * MS + B];
                        }
                }
                if constexpr (TM >= 2)   // filter pairs FP[a][b] = (kf_0[a][b], kf_1[a][b])
                    for (int a2 = 0; a2 < MS; ++a2)
                        for (int b2 = 0; b2 < MS; ++b2)
                            grp[2 * (a2 * MS + b2) + fi] = k[(MS - 1 - a2) * MS + (MS - 1 - b2)];
            }
        }
    }

    // one launch per stage as clusters of `cl` CTAs per tile (stage_kernel_cl*:
    // the cluster's CTAs split the tile's filter groups and sum their partial
    // forces in rank order through distributed shared memory)
    static int launch_cluster(const StageArgs& a, int batch, int cl, cudaStream_t s,
                              const float* htaps = nullptr) {
        int dev = 0;
        cudaGetDevice(&dev);
        StageArgs b = a;
        const int tiles_x = (a.W + TW - 1) / TW, tiles_y = (a.H + TH - 1) / TH;
        if ((long)tiles_x * tiles_y > 65535) return fail(TNRD_EUNSUPPORTED, "cluster kernel: too many tiles per image");
        const dim3 grid(cl, tiles_x * tiles_y, batch);
        auto set_groups = [&](int ng) {
            b.ngroups = ng;
            b.cluster = cl;
            b.cl_gper = ng / cl;
            b.cl_gextra = ng % cl;
            b.cl_tiles_x = tiles_x;
        };
        if constexpr (kPT) {
            if (htaps && pt_fits(a)) {
                static std::mutex mu2;
                static uint64_t attr2 = 0;
                auto kern = stage_kernel_cl_pt<MS, TH, TW, RF_PT, RB, NT, FAST, F_TILE_PT, TNRD_PT_TILE_MINB, TB, kTmCluster>;
                int rc = prepare(kern, dev, attr2, mu2);
                if (rc) return rc;
                TB tb;
                fill_taps<kTmCluster, F_TILE_PT>(tb, htaps, a.nk);
                set_groups((a.nk + F_TILE_PT - 1) / F_TILE_PT);
                CUDA_TRY(launch_pdl_cluster(kern, grid, NT, pt_smem<CPT, F_TILE_PT>(a), cl, s, b, tb));
                g_launches.fetch_add(1);
                return TNRD_OK;
            }
        }
        static std::mutex mu;
        static uint64_t attr_set = 0;  // per-device bitmask
        auto kern = stage_kernel_cl<MS, TH, TW, RF, RB, NT, FAST, F, MINB>;
        int rc = prepare(kern, dev, attr_set, mu);
        if (rc) return rc;
        set_groups((a.nk + F - 1) / F);
        CUDA_TRY(launch_pdl_cluster(kern, grid, NT, C::smem_bytes(a.tab_stride), cl, s, b));
        g_launches.fetch_add(1);
        return TNRD_OK;
    }
    // filter groups of the cluster kernel for this model (the cluster size
    // never exceeds it)
    static int cluster_groups(const StageArgs& a) {
        if constexpr (kPT)
            if (pt_fits(a)) return (a.nk + F_TILE_PT - 1) / F_TILE_PT;
        return (a.nk + F - 1) / F;
    }

    static int launch(const StageArgs& a, int batch, cudaStream_t s, const float* htaps = nullptr) {
        static std::mutex mu;
        static uint64_t attr_set = 0;  // per-device bitmask
        int dev = 0;
        cudaGetDevice(&dev);
        StageArgs b = a;
        b.ngroups = (a.nk + F - 1) / F;
        const dim3 grid((a.W + TW - 1) / TW, (a.H + TH - 1) / TH, batch);
        if constexpr (kPT) {
            if (htaps && pt_fits(a)) {
                static std::mutex mu2;
                static uint64_t attr2 = 0;
                auto kern = stage_kernel_pt<MS, TH, TW, RF_PT, RB, NT, FAST, F_TILE_PT, TNRD_PT_TILE_MINB, TB, kTmTile>;
                int rc = prepare(kern, dev, attr2, mu2);
                if (rc) return rc;
                TB tb;
                fill_taps<kTmTile, F_TILE_PT>(tb, htaps, a.nk);
                b.ngroups = (a.nk + F_TILE_PT - 1) / F_TILE_PT;
                CUDA_TRY(launch_pdl(kern, grid, NT, pt_smem<CPT, F_TILE_PT>(a), s, b, tb));
                g_launches.fetch_add(1);
                return TNRD_OK;
            }
        }
        auto kern = stage_kernel<MS, TH, TW, RF, RB, NT, FAST, F, MINB>;
        int rc = prepare(kern, dev, attr_set, mu);
        if (rc) return rc;
        CUDA_TRY(launch_pdl(kern, grid, NT, C::smem_bytes(a.tab_stride), s, b));
        g_launches.fetch_add(1);
        return TNRD_OK;
    }

#ifdef TNRD_EXPERIMENTS
    // all T stages in one persistent dataflow launch (+ the setup kernel)
    static int launch_fused(const tnrd_model* md, const StageArgs* st, int nst, int batch,
                            cudaStream_t s) {
        const int T_ = nst;
        static std::mutex mu;
        static uint64_t attr_set = 0;
        static int occ[64] = {0};
        const size_t smem = C::smem_bytes(st[0].tab_stride);
        int dev = 0;
        cudaGetDevice(&dev);
        auto kern = fused::despeckle_fused_kernel<MS, TH, TW, RF, RB, NT, FAST, F, MINB>;
        int rc = prepare(kern, dev, attr_set, mu);
        if (rc) return rc;
        int per_sm = 0;
        {
            std::lock_guard<std::mutex> lk(mu);
            per_sm = occ[dev & 63];
            if (per_sm == 0) {
                CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
                occ[dev & 63] = per_sm = std::max(per_sm, 1);
            }
        }
        const int ng = (st[0].nk + F - 1) / F;
        const int tiles_x = (st[0].W + TW - 1) / TW, tiles_y = (st[0].H + TH - 1) / TH;
        const int tiles = tiles_x * tiles_y * batch;
        const int grid = std::min(sm_count() * per_sm, T_ * tiles * ((ng + kFusedClaim - 1) / kFusedClaim));
        const std::vector<long> key = {tiles_x, tiles_y, tiles, T_, ng, grid, MS, TH};
        void* wsp = nullptr;
        FusedLayout L;
        rc = fused_workspace(md, s, key, T_, tiles, tiles_x, ng, TH * TW, grid, &wsp, &L);
        if (rc) return rc;
        char* base = static_cast<char*>(wsp);
        FusedSetup su;
        su.T = T_;
        su.dst = reinterpret_cast<StageArgs*>(base + L.stargs);
        for (int t = 0; t < T_; ++t) {
            su.st[t] = st[t];
            su.st[t].ngroups = ng;
        }
        fused_setup_kernel<<<1, 32, 0, s>>>(su);
        CUDA_TRY(cudaGetLastError());
        fused::FusedArgs fa;
        fa.st = su.dst;
        fa.seq = reinterpret_cast<const int*>(base + L.seq);
        fa.nclaims = L.nclaims;
        fa.T = T_;
        fa.claim_groups = kFusedClaim;
        fa.part0 = reinterpret_cast<float*>(base + L.part0);
        fa.part1 = reinterpret_cast<float*>(base + L.part1);
        fa.ctl = reinterpret_cast<uint32_t*>(base + L.ctl);
        fa.cnt = fa.ctl + 2;
        fa.done = fa.cnt + (size_t)T_ * tiles;
        fa.tiles_x = tiles_x;
        fa.tiles_y = tiles_y;
        fa.tiles = tiles;
        kern<<<grid, NT, smem, s>>>(fa);
        CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(2);
        return TNRD_OK;
    }

#endif  // TNRD_EXPERIMENTS

    static long tiles(const StageArgs& a, int batch) {
        return (long)((a.W + TW - 1) / TW) * ((a.H + TH - 1) / TH) * batch;
    }
    static size_t ws_bytes(const StageArgs& a, int batch) {
        const long nt = tiles(a, batch);
        const int fs = split_f(a);
        return (size_t)nt * ((a.nk + fs - 1) / fs) * TH * TW * sizeof(float);
    }

    // persistent grid of (SMs x resident CTAs) over (tile, group) units
    static int launch_split(const StageArgs& a, int batch, void* wsp, cudaStream_t s,
                            const float* htaps = nullptr) {
        if constexpr (kPT) {
            if (htaps && pt_fits(a)) {
                static std::mutex mu;
                static uint64_t attr_set = 0;
                static int occ[64] = {0};
                auto kern = stage_kernel_split_pt<MS, TH, TW, RF_SPLIT_PT, RB, NT, FAST, F_SPLIT_PT, TNRD_PT_MINB, TB,
                                                  kTmSplit>;
                TB tb;
                fill_taps<kTmSplit, F_SPLIT_PT>(tb, htaps, a.nk);
                return launch_split_k(kern, pt_smem<CPS, F_SPLIT_PT>(a), F_SPLIT_PT, a, batch, wsp, s, mu,
                                      attr_set, occ, tb);
            }
        }
        static std::mutex mu;
        static uint64_t attr_set = 0;
        static int occ[64] = {0};
        auto kern = stage_kernel_split<MS, TH, TW, RF, RB, NT, FAST, F, MINB>;
        return launch_split_k(kern, C::smem_bytes(a.tab_stride), F, a, batch, wsp, s, mu, attr_set, occ);
    }

    template <class K, class... Extra>
    static int launch_split_k(K kern, size_t smem, int fgroup, const StageArgs& a, int batch, void* wsp,
                              cudaStream_t s, std::mutex& mu, uint64_t& attr_set, int* occ,
                              const Extra&... extra) {
        int dev = 0;
        cudaGetDevice(&dev);
        int rc = prepare(kern, dev, attr_set, mu);
        if (rc) return rc;
        int per_sm = 0, sms = 0;
        {
            std::lock_guard<std::mutex> lk(mu);
            per_sm = occ[dev & 63];
            if (per_sm == 0) {
                CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
                occ[dev & 63] = per_sm = std::max(per_sm, 1);
            }
        }
        CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        StageArgs b = a;
        b.ngroups = (a.nk + fgroup - 1) / fgroup;
        SplitWs w;
        w.tiles_x = (a.W + TW - 1) / TW;
        w.tiles_y = (a.H + TH - 1) / TH;
        w.tiles = w.tiles_x * w.tiles_y * batch;
        w.part = reinterpret_cast<float*>(static_cast<char*>(wsp) + kSplitCtlBytes);
        const long units = (long)w.tiles * b.ngroups;
        const int grid = (int)std::min<long>(units, (long)sms * per_sm);
        // SM-aware ranges (tnrd_stage.cuh SplitWs) for the parameter-space
        // kernel when the grid is whole SMs x resident CTAs
        w.ctl = static_cast<uint32_t*>(wsp);
        w.map_sms = (kMapSplit && sizeof...(extra) > 0 && grid % sms == 0 && sms <= kSplitCtlSms &&
                     grid <= kSplitCtlRanges) ? sms : 0;
        CUDA_TRY(launch_pdl(kern, grid, NT, smem, s, b, w, extra...));
        const long quads = (long)w.tiles * (TH * TW / 4);
        const int rgrid = (int)std::min<long>((quads + 127) / 128, (long)sms * 16);
        CUDA_TRY(launch_pdl(stage_reduce_kernel<TH, TW>, rgrid, 128, 0, s, b, w));
        g_launches.fetch_add(2);
        return TNRD_OK;
    }
};

// Kernel choice (measured on B200): whole large tiles once
// the grid gives >= 3 waves of 2 CTAs per SM; below that the split kernel,
// with large tiles when there are >= 2 units per CTA slot, else small tiles
// (more, cheaper units: a 256^2 image).
static int sm_count() {
    static std::atomic<int> cached{0};
    int n = cached.load();
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached.store(n);
    }
    return n;
}

static bool use_large_tiles(const StageArgs& a, int batch) {
    return StageKernel<7, true, LargeTile>::tiles(a, batch) >= 3L * 2 * sm_count();
}

static bool use_split_large(const StageArgs& a, int batch) {
    const long units = StageKernel<7, true, SplitTile>::tiles(a, batch) * ((a.nk + SplitTile::F - 1) / SplitTile::F);
    return units >= 2L * 2 * sm_count();
}

// CTAs per cluster for a grid of `tiles` large / small tiles with `groups`
// filter groups on `slots` resident CTA slots (measured on B200,
// tools/grid_sweep.py, profiles/r02_cluster): 2 once two CTAs per tile give
// >= 3.4 waves (finer CTAs only add staging and cluster barriers), else 4
// while that fills 3/4 of a wave, else the largest cluster (<= 8) that fits
// one wave.  A forced size (tnrd_set_cluster_size / TNRD_CLUSTER_SIZE) wins.
static int cluster_size(long tiles, int groups, long slots) {
    int forced = g_cluster_size.load();
    if (forced == 0) {
        static const int env = [] {
            const char* e = std::getenv("TNRD_CLUSTER_SIZE");
            const int v = e ? std::atoi(e) : 0;
            return (v >= 2 && v <= kMaxCluster) ? v : 0;
        }();
        forced = env;
    }
    groups = std::max(groups, 1);
    if (forced) return std::min(forced, groups);
    tiles = std::max(tiles, 1L);
    long cl;
    if (10 * 2 * tiles >= 34 * slots) cl = 2;
    else if (4 * 4 * tiles >= 3 * slots) cl = 4;
    else cl = std::min<long>(kMaxCluster, std::max<long>(slots / tiles, 2));
    return (int)std::min<long>(cl, groups);
}

// Auto mode (measured on B200, profiles/r02_cluster/grid_sweep_*.txt): the
// tile kernel from 6 waves of large tiles (2 x 3 waves: the batch fork's two
// halves, or one big scene); below that the cluster kernel -- one launch per
// stage, a tile's filter groups on 2..8 CTAs -- with large tiles when there
// are >= 2 (tile, group) units per CTA slot, else small tiles (a 256^2
// image).  The split kernel (two launches per stage) is no longer chosen
// (TNRD_AUTO_CLUSTER=0 restores it); a thread-local override pins the
// variant where two launches must agree bit for bit (the batch fork's
// halves, the scene bands).
#ifndef TNRD_AUTO_CLUSTER
#define TNRD_AUTO_CLUSTER 1
#endif
static bool auto_cluster() {
    static const bool on = [] {
        const char* e = std::getenv("TNRD_AUTO_CLUSTER");
        return e ? e[0] != '0' : (TNRD_AUTO_CLUSTER != 0);
    }();
    return on;
}
static thread_local int t_force_variant = -1;
struct VariantGuard {
    int prev;
    explicit VariantGuard(int v) : prev(t_force_variant) { t_force_variant = v; }
    ~VariantGuard() { t_force_variant = prev; }
};

// tile configuration of the CUDA-core stage for this launch: 0 tile kernel
// small tiles, 1 tile kernel large tiles, 2 split kernel large, 3 split
// small, 4 cluster kernel large tiles, 5 cluster kernel small tiles
static int cc_variant(const StageArgs& a, int batch) {
    switch (g_kernel_mode.load()) {
        case 3: return 0;
        case 4: return 1;
        case 6: return 2;
        case 7: return 3;
        case 10: return 4;
        case 11: return 5;
        default:
            if (t_force_variant >= 0) return t_force_variant;
            if (!auto_cluster())
                return use_large_tiles(a, batch) ? 1 : (use_split_large(a, batch) ? 2 : 3);
            if (StageKernel<7, true, LargeTile>::tiles(a, batch) >= 2 * 3L * 2 * sm_count()) return 1;
            return use_split_large(a, batch) ? 4 : 5;
    }
}

template <bool FAST, class T>
static int dispatch_m_t(int m, const StageArgs& a, int batch, cudaStream_t s, const float* htaps = nullptr) {
    switch (m) {
        case 3: return StageKernel<3, FAST, T>::launch(a, batch, s, htaps);
        case 5: return StageKernel<5, FAST, T>::launch(a, batch, s, htaps);
        case 7: return StageKernel<7, FAST, T>::launch(a, batch, s, htaps);
        case 9: return StageKernel<9, FAST, T>::launch(a, batch, s, htaps);
        default: return fail(TNRD_EUNSUPPORTED, "unsupported filter size %d", m);
    }
}

template <bool FAST, class T>
static int dispatch_cluster_m_t(int m, const StageArgs& a, int batch, long slots_per_sm, cudaStream_t s,
                                const float* htaps = nullptr) {
    const long slots = slots_per_sm * sm_count();
    switch (m) {
        case 3: { using K = StageKernel<3, FAST, T>;
                  return K::launch_cluster(a, batch, std::max(2, cluster_size(K::tiles(a, batch), K::cluster_groups(a), slots)), s, htaps); }
        case 5: { using K = StageKernel<5, FAST, T>;
                  return K::launch_cluster(a, batch, std::max(2, cluster_size(K::tiles(a, batch), K::cluster_groups(a), slots)), s, htaps); }
        case 7: { using K = StageKernel<7, FAST, T>;
                  return K::launch_cluster(a, batch, std::max(2, cluster_size(K::tiles(a, batch), K::cluster_groups(a), slots)), s, htaps); }
        case 9: { using K = StageKernel<9, FAST, T>;
                  return K::launch_cluster(a, batch, std::max(2, cluster_size(K::tiles(a, batch), K::cluster_groups(a), slots)), s, htaps); }
        default: return fail(TNRD_EUNSUPPORTED, "unsupported filter size %d", m);
    }
}

template <bool FAST, class T>
static size_t split_bytes_m_t(int m, const StageArgs& a, int batch) {
    switch (m) {
        case 3: return StageKernel<3, FAST, T>::ws_bytes(a, batch);
        case 5: return StageKernel<5, FAST, T>::ws_bytes(a, batch);
        case 7: return StageKernel<7, FAST, T>::ws_bytes(a, batch);
        default: return StageKernel<9, FAST, T>::ws_bytes(a, batch);
    }
}

template <bool FAST, class T>
static int dispatch_split_m_t(int m, const StageArgs& a, int batch, void* ws, cudaStream_t s,
                              const float* htaps = nullptr) {
    switch (m) {
        case 3: return StageKernel<3, FAST, T>::launch_split(a, batch, ws, s, htaps);
        case 5: return StageKernel<5, FAST, T>::launch_split(a, batch, ws, s, htaps);
        case 7: return StageKernel<7, FAST, T>::launch_split(a, batch, ws, s, htaps);
        case 9: return StageKernel<9, FAST, T>::launch_split(a, batch, ws, s, htaps);
        default: return fail(TNRD_EUNSUPPORTED, "unsupported filter size %d", m);
    }
}

// the stream's split workspace, grown on demand (outside stream capture)
static int split_workspace(const tnrd_model* md, cudaStream_t s, size_t part_bytes, void** out) {
    std::lock_guard<std::mutex> lk(md->ws_mu);
    auto& b = md->ws[s];
    const size_t bytes = split_alloc_bytes(part_bytes);
    if (b.bytes < bytes) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(s, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            return fail(TNRD_ECUDA, "split workspace must be allocated before stream capture");
        if (b.ptr) {
            md->retired.push_back(b.ptr);   // a captured graph may still use it
            b.ptr = nullptr;
            b.bytes = 0;
        }
        CUDA_TRY(cudaMalloc(&b.ptr, bytes));
        b.bytes = bytes;
        // control words start zeroed (the kernels leave them zeroed); the
        // partials region may be reused by other sizes, the control words
        // sit past the largest partials this buffer holds
        CUDA_TRY(cudaMemsetAsync(b.ptr, 0, bytes, s));
    }
    *out = b.ptr;
    return TNRD_OK;
}

template <bool FAST>
static int dispatch_m(const tnrd_model* md, const StageArgs& a, int batch, cudaStream_t s) {
    const int m = md->m;
    const int v = cc_variant(a, batch);
    const float* htaps = md->h_taps.data() + (size_t)a.stage * md->nk_pad * md->kp;
    if (v == 0) return dispatch_m_t<FAST, SmallTile>(m, a, batch, s);
    if (v == 1) return dispatch_m_t<FAST, LargeTile>(m, a, batch, s, htaps);
    if (v == 4) return dispatch_cluster_m_t<FAST, LargeTile>(m, a, batch, 2, s, htaps);
    if (v == 5) return dispatch_cluster_m_t<FAST, SmallTile>(m, a, batch, m >= 9 ? 2 : 3, s);
    // the split kernel's partials workspace is bounded (it only pays off on
    // small grids anyway)
    if ((v == 2 ? split_bytes_m_t<FAST, SplitTile>(m, a, batch)
                : split_bytes_m_t<FAST, SmallTile>(m, a, batch)) > kMaxSplitBytes)
        return dispatch_m_t<FAST, LargeTile>(m, a, batch, s, htaps);
    const size_t bytes = v == 2 ? split_bytes_m_t<FAST, SplitTile>(m, a, batch)
                                : split_bytes_m_t<FAST, SmallTile>(m, a, batch);
    void* ws = nullptr;
    int rc = split_workspace(md, s, bytes, &ws);
    if (rc) return rc;
    return v == 2 ? dispatch_split_m_t<FAST, SplitTile>(m, a, batch, ws, s, htaps)
                  : dispatch_split_m_t<FAST, SmallTile>(m, a, batch, ws, s);
}

#ifdef TNRD_EXPERIMENTS
template <int MS>
struct StageKernelTC {
    using C = tc::TcCfg<MS>;
    // two CTAs per SM (TMEM: 2 x 256 columns)
    static bool fits(int tab_stride) { return C::smem_bytes(tab_stride) <= 112 * 1024; }
    static int launch(const StageArgs& a, const float* bop, int batch, cudaStream_t s) {
        static std::mutex mu;
        static uint64_t attr_set = 0;
        const size_t smem = C::smem_bytes(a.tab_stride);
        int dev = 0;
        cudaGetDevice(&dev);
        auto kern = tc::stage_kernel_tc<MS>;
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!(attr_set & (1ull << (dev & 63)))) {
                CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              112 * 1024));
                attr_set |= 1ull << (dev & 63);
            }
        }
        dim3 grid((a.W + C::TW - 1) / C::TW, (a.H + C::TH - 1) / C::TH, batch);
        kern<<<grid, tc::kNT, smem, s>>>(a, bop);
        CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1);
        return TNRD_OK;
    }
};

template <int MS>
struct StageKernelTC3 {
    using C = tc3::Cfg<MS>;
    static bool fits(int tab_stride) { return C::smem_bytes(tab_stride) <= 227 * 1024; }
    static int launch(const StageArgs& a, const float* bop, int batch, cudaStream_t s) {
        static std::mutex mu;
        static uint64_t attr_set = 0;
        const size_t smem = C::smem_bytes(a.tab_stride);
        int dev = 0;
        cudaGetDevice(&dev);
        auto kern = tc3::stage_kernel_tc3<MS>;
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!(attr_set & (1ull << (dev & 63)))) {
                CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              227 * 1024));
                attr_set |= 1ull << (dev & 63);
            }
        }
        dim3 grid((a.W + C::TW - 1) / C::TW, (a.H + C::TH - 1) / C::TH, batch);
        kern<<<grid, tc3::kNT, smem, s>>>(a, bop);
        CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1);
        return TNRD_OK;
    }
};

static bool tc3_supported(const tnrd_model* md) {
    if (!md->fast || !md->d_bop) return false;
    switch (md->m) {
        case 3: return StageKernelTC3<3>::fits(md->tab_stride);
        case 5: return StageKernelTC3<5>::fits(md->tab_stride);
        case 7: return StageKernelTC3<7>::fits(md->tab_stride);
        default: return false;
    }
}

static int dispatch_tc3(const tnrd_model* md, int t, StageArgs a, int batch, cudaStream_t s) {
    a.ngroups = md->nk_pad / tc::kG;
    const float* bop = md->d_bop + (size_t)t * md->bop_stage;
    switch (md->m) {
        case 3: return StageKernelTC3<3>::launch(a, bop, batch, s);
        case 5: return StageKernelTC3<5>::launch(a, bop, batch, s);
        case 7: return StageKernelTC3<7>::launch(a, bop, batch, s);
        default: return fail(TNRD_EUNSUPPORTED, "no tensor-core stage kernel for m=%d", md->m);
    }
}

static bool tc_supported(const tnrd_model* md) {
    if (!md->fast || !md->d_bop) return false;
    switch (md->m) {
        case 3: return StageKernelTC<3>::fits(md->tab_stride);
        case 5: return StageKernelTC<5>::fits(md->tab_stride);
        case 7: return StageKernelTC<7>::fits(md->tab_stride);
        case 9: return StageKernelTC<9>::fits(md->tab_stride);
        default: return false;
    }
}

static int dispatch_tc(const tnrd_model* md, int t, StageArgs a, int batch, cudaStream_t s) {
    a.ngroups = md->nk_pad / tc::kG;
    const float* bop = md->d_bop + (size_t)t * md->bop_stage;
    switch (md->m) {
        case 3: return StageKernelTC<3>::launch(a, bop, batch, s);
        case 5: return StageKernelTC<5>::launch(a, bop, batch, s);
        case 7: return StageKernelTC<7>::launch(a, bop, batch, s);
        case 9: return StageKernelTC<9>::launch(a, bop, batch, s);
        default: return fail(TNRD_EUNSUPPORTED, "no tensor-core stage kernel for m=%d", md->m);
    }
}


// ---- z-field stage (tnrd_stage_zf.cuh): tcgen05 forward -> z planes, then
// TMA-fed RBF + adjoint + prox ------------------------------------------------

#ifndef TNRD_ZF_PASSES
#define TNRD_ZF_PASSES 6
#endif
static std::atomic<int> g_zf_passes{TNRD_ZF_PASSES};

extern "C" int tnrd_set_zfield_passes(int n) {
    if (n != 3 && n != 4 && n != 6) return fail(TNRD_EINVAL, "z-field pass count must be 3, 4 or 6");
    g_zf_passes.store(n);
    return TNRD_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static std::atomic<PFN_cuTensorMapEncodeTiled_v12000> fn{nullptr};
    PFN_cuTensorMapEncodeTiled_v12000 f = fn.load();
    if (!f) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        fn.store(f);
    }
    return f;
}

// z-stage tile configurations: large tiles for batches / big scenes, small
// tiles (half height) when the grid would not fill the SMs; both keep one
// filter split (NSPLIT = 1), so the per-pixel summation order -- and the
// result bits -- do not depend on the choice
struct ZTileL { static constexpr int TH = 64, TW = 64, RB = 4, NT = 256, F = 2, MINB = 2; };
struct ZTileS { static constexpr int TH = 32, TW = 64, RB = 2, NT = 256, F = 2, MINB = 2; };

template <int MS, int NP>
static int launch_zfield(const zf::ZArgs& z, int gx, int gy, int batch, cudaStream_t s) {
    using C = zf::ZCfg<MS, NP>;
    static std::mutex mu;
    static uint64_t attr_set = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = zf::zfield_kernel<MS, NP>;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!(attr_set & (1ull << (dev & 63)))) {
            CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)C::smem_bytes()));
            attr_set |= 1ull << (dev & 63);
        }
    }
    CUDA_TRY(launch_pdl(kern, dim3(gx, gy, batch), zf::kZThreads, C::smem_bytes(), s, z));
    return TNRD_OK;
}

template <int MS, class T>
static int launch_zstage(const zf::ZStageArgs& za, const CUtensorMap& map, int batch, cudaStream_t s) {
    using C = zf::ZSCfg<MS, T::TH, T::TW, T::RB, T::NT, T::F>;
    static std::mutex mu;
    static uint64_t attr_set = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = zf::zstage_kernel<MS, T::TH, T::TW, T::RB, T::NT, T::F, T::MINB>;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!(attr_set & (1ull << (dev & 63)))) {
            CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr_set |= 1ull << (dev & 63);
        }
    }
    const size_t smem = C::smem_bytes(za.s.tab_stride);
    dim3 grid((za.s.W + T::TW - 1) / T::TW, (za.s.H + T::TH - 1) / T::TH, batch);
    CUDA_TRY(launch_pdl(kern, grid, T::NT, smem, s, za, map));
    return TNRD_OK;
}

template <int MS>
static int dispatch_zfield_np(int np, const zf::ZArgs& z, int gx, int gy, int batch, cudaStream_t s) {
    switch (np) {
        case 16: return launch_zfield<MS, 16>(z, gx, gy, batch, s);
        case 32: return launch_zfield<MS, 32>(z, gx, gy, batch, s);
        case 48: return launch_zfield<MS, 48>(z, gx, gy, batch, s);
        case 64: return launch_zfield<MS, 64>(z, gx, gy, batch, s);
        case 80: return launch_zfield<MS, 80>(z, gx, gy, batch, s);
        case 96: return launch_zfield<MS, 96>(z, gx, gy, batch, s);
        case 112: return launch_zfield<MS, 112>(z, gx, gy, batch, s);
        case 128: return launch_zfield<MS, 128>(z, gx, gy, batch, s);
        default: return fail(TNRD_EUNSUPPORTED, "z-field kernel: nk_pad %d", np);
    }
}

template <class T>
static int dispatch_zstage_m(int m, const zf::ZStageArgs& za, const CUtensorMap& map, int batch,
                             cudaStream_t s) {
    switch (m) {
        case 3: return launch_zstage<3, T>(za, map, batch, s);
        case 5: return launch_zstage<5, T>(za, map, batch, s);
        case 7: return launch_zstage<7, T>(za, map, batch, s);
        default: return fail(TNRD_EUNSUPPORTED, "z-field stage: m=%d", m);
    }
}

static bool zf_supported(const tnrd_model* md) {
    return md->fast && md->d_zop && md->m <= 7 && md->nk_pad <= 128 && tensor_map_encoder() != nullptr;
}

static int launch_zf(const tnrd_model* md, int t, const StageArgs& a, int batch, cudaStream_t s) {
    const int m = md->m, R = m / 2, np = md->nk_pad;
    const bool top_halo = a.flags & TNRD_STAGE_TOP_HALO, bot_halo = a.flags & TNRD_STAGE_BOTTOM_HALO;
    const int64_t zld = round_up(a.W + 2 * R, 4);   // plane column = image column + r
    const int64_t zrows = a.H + 2 * R;
    const int64_t zplane = zrows * zld;
    const size_t bytes = (size_t)batch * np * zplane * sizeof(float);
    // the stream's z planes, grown on demand (outside capture)
    float* zbuf = nullptr;
    {
        std::lock_guard<std::mutex> lk(md->ws_mu);
        auto& b = md->zws[s];
        if (b.bytes < bytes) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            CUDA_TRY(cudaStreamIsCapturing(s, &cs));
            if (cs != cudaStreamCaptureStatusNone)
                return fail(TNRD_ECUDA, "z-field workspace must be allocated before stream capture");
            if (b.ptr) {
                md->retired.push_back(b.ptr);   // a captured graph may still use it
                b.ptr = nullptr;
                b.bytes = 0;
            }
            CUDA_TRY(cudaMalloc(&b.ptr, bytes));
            b.bytes = bytes;
        }
        zbuf = static_cast<float*>(b.ptr);
    }
    zf::ZArgs z;
    z.u_in = a.u_in; z.ld = a.ld; z.img_stride = a.img_stride;
    z.H = a.H; z.W = a.W;
    z.flags = a.flags & (TNRD_STAGE_FLOOR_INPUT | TNRD_STAGE_TOP_HALO | TNRD_STAGE_BOTTOM_HALO);
    z.u0_floor = a.u0_floor;
    z.bop = md->d_zop + (size_t)t * md->zop_stage;
    z.z = zbuf; z.zld = zld; z.zplane = zplane; z.zimg = np * zplane;
    z.zrow0 = top_halo ? -R : 0;
    z.zrow_end = bot_halo ? a.H + R : a.H;
    const int np_ = g_zf_passes.load();
    // (u piece, k piece) products, largest first
    static const int pu6[6] = {0, 1, 0, 2, 1, 0}, pk6[6] = {0, 0, 1, 0, 1, 2};
    static const int pu4[4] = {0, 1, 0, 1}, pk4[4] = {0, 0, 1, 1};
    const int* pu = np_ == 4 ? pu4 : pu6;
    const int* pk = np_ == 4 ? pk4 : pk6;
    z.npass = np_;
    z.pass_u = 0; z.pass_k = 0;
    for (int i = 0; i < np_; ++i) {
        z.pass_u |= (uint32_t)pu[i] << (2 * i);
        z.pass_k |= (uint32_t)pk[i] << (2 * i);
    }
    const int gx = (a.W + R + zf::kBandCols - 1) / zf::kBandCols;   // bands start at 32 bx - r
    const int gy = (z.zrow_end - z.zrow0 + zf::kBandRows - 1) / zf::kBandRows;
    int rc = TNRD_OK;
    switch (m) {
        case 3: rc = dispatch_zfield_np<3>(np, z, gx, gy, batch, s); break;
        case 5: rc = dispatch_zfield_np<5>(np, z, gx, gy, batch, s); break;
        case 7: rc = dispatch_zfield_np<7>(np, z, gx, gy, batch, s); break;
        default: return fail(TNRD_EUNSUPPORTED, "z-field kernel: m=%d", m);
    }
    if (rc) return rc;
    static const int zf_debug = getenv("TNRD_ZF_DEBUG") ? atoi(getenv("TNRD_ZF_DEBUG")) : 0;
    if (zf_debug == 1) return TNRD_OK;   // zfield only
    if (zf_debug == 2) {
        CUDA_TRY(cudaStreamSynchronize(s));
        fprintf(stderr, "zf debug: zfield ok\n");
    }

    const bool large = (long)((a.W + 63) / 64) * ((a.H + 63) / 64) * batch >= 2L * sm_count();
    const int F = large ? ZTileL::F : ZTileS::F;
    const int TH = large ? ZTileL::TH : ZTileS::TH, TW = large ? ZTileL::TW : ZTileS::TW;
    CUtensorMap map;
    {
        const cuuint64_t dims[3] = {(cuuint64_t)zld, (cuuint64_t)zrows, (cuuint64_t)batch * np};
        const cuuint64_t strides[2] = {(cuuint64_t)zld * 4, (cuuint64_t)zplane * 4};
        const cuuint32_t box[3] = {(cuuint32_t)round_up(TW + 2 * R, 4), (cuuint32_t)(TH + 2 * R), (cuuint32_t)F};
        const cuuint32_t es[3] = {1, 1, 1};
        CUresult r = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, zbuf, dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(TNRD_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    zf::ZStageArgs za;
    za.s = a;
    za.s.ngroups = (md->nk + F - 1) / F;
    za.np = np;
    rc = large ? dispatch_zstage_m<ZTileL>(m, za, map, batch, s) : dispatch_zstage_m<ZTileS>(m, za, map, batch, s);
    if (rc) return rc;
    if (zf_debug == 2) {
        CUDA_TRY(cudaStreamSynchronize(s));
        fprintf(stderr, "zf debug: zstage ok\n");
    }
    g_launches.fetch_add(2);
    return TNRD_OK;
}


#else
extern "C" int tnrd_set_zfield_passes(int n) {
    (void)n;
    return fail(TNRD_EUNSUPPORTED, "z-field kernel not built (TNRD_EXPERIMENTS)");
}

#endif  // TNRD_EXPERIMENTS

static int check_shape(const tnrd_model* md, int batch, int H, int W, int64_t ld,
                       int64_t image_stride) {
    if (batch < 1 || batch > 65535) return fail(TNRD_EINVAL, "batch must be in [1, 65535], got %d", batch);
    if (H < 1 || W < 1) return fail(TNRD_EINVAL, "image must have at least one pixel");
    if (md->m > 2 * std::min(H, W) + 1)
        return fail(TNRD_EINVAL, "kernel size %d degenerate for image of shape (%d, %d)", md->m, H, W);
    if (ld < W) return fail(TNRD_EINVAL, "row stride %lld < width %d", (long long)ld, W);
    if (batch > 1 && image_stride < ld * H)
        return fail(TNRD_EINVAL, "image stride %lld too small", (long long)image_stride);
    return TNRD_OK;
}

// stage t's kernel arguments (model tables, RBF and reaction constants)
static StageArgs stage_args(const tnrd_model* md, int t, uint32_t flags) {
    StageArgs a;
    a.u_in = nullptr; a.f = nullptr; a.u_out = nullptr;
    a.taps = md->d_taps + (size_t)t * md->nk_pad * md->kp;
    a.tab = md->d_tab + (size_t)t * md->nk_pad * md->tab_stride;
    a.ld = 0; a.img_stride = 0;
    a.H = 0; a.W = 0;
    a.ngroups = round_up(md->nk, kF) / kF;
    a.nk = md->nk;
    a.tab_stride = md->tab_stride;
    const double lam = md->lam[t];
    const double aa = 1.0 + 2.0 * lam;
    a.lam4 = (float)(4.0 * lam);
    a.c8 = (float)(8.0 * aa * lam);
    a.inv2a = (float)(1.0 / (2.0 * aa));
    const double L2E = 1.4426950408889634;
    a.inv_h = (float)(1.0 / md->h);
    a.tab_bias = 0u - (0x4B400000u << 5);
    a.tab_ni = md->nip;
    a.t_off = (float)(1.0 - md->zlo / md->h);
    a.tmax = (float)(md->ni + 1);
    a.tab3 = md->tab3_stride ? md->d_tab3 + (size_t)t * md->nk_pad * md->tab3_stride : nullptr;
    a.tab3_stride = md->tab3_stride;
    a.tab3_bias = 0u - (0x4B400000u << 4);
    a.inv_h3 = md->tab3_stride ? (float)(1.0 / md->h3) : 0.0f;
    a.t_off3 = md->tab3_stride ? (float)(1.0 - md->zlo / md->h3) : 0.0f;
    a.tmax3 = (float)(md->ni3 + 1);
    a.delta = (float)md->delta;
    a.cE = (float)(-L2E / (2.0 * md->gamma * md->gamma));
    a.mu0 = (float)md->mu0;
    a.M = md->M;
    a.lam = (float)lam;
    a.pfloor = (float)md->floor;
    a.tau = (float)(0.01 * md->floor);       // PROJECTION_KNEE (diffusion.py:24)
    a.inv_tau = (float)(1.0 / (0.01 * md->floor));
    a.u0_floor = md->variant == TNRD_VARIANT_PROJECTED ? (float)md->floor : kFFloor;
    if (md->variant == TNRD_VARIANT_PROJECTED) flags |= TNRD_STAGE_PROJECTED;
    a.flags = flags;
    a.stage = t;
    a.status = nullptr;
    a.force_out = nullptr;
    a.cluster = 1; a.cl_gper = 0; a.cl_gextra = 0; a.cl_tiles_x = 1;
    return a;
}


// ---- tensor-core adjoint stage (tnrd_stage_adj.cuh, mode 12) ---------------
// B operand of the adjoint GEMM psi = Phi K^T for every stage: K-major
// [ks][prec][kc][n][e] = piece_prec(k_i[n]), i = 8 ks + 4 kc + e, n = the tap
// index a m + b of the reference kernel k_i (zero for n >= m^2, i >= nk);
// prec 0 = tf32 rna(k), 1 = rna(k - hi).
static int adj_operand(const tnrd_model* md, int nb, int kc) {
    std::lock_guard<std::mutex> lk(md->ws_mu);
    if (md->d_aop) return TNRD_OK;
    const int ks = kc / 2, mm = md->m * md->m;
    const size_t per_stage = (size_t)ks * 2 * 2 * nb * 4;
    std::vector<float> h((size_t)md->T * per_stage, 0.0f);
    for (int t = 0; t < md->T; ++t)
        for (int i = 0; i < md->nk; ++i) {
            const float* k = md->h_taps.data() + ((size_t)t * md->nk_pad + i) * md->kp;
            const int s8 = i / 8, c2 = (i % 8) / 4, e = i % 4;
            for (int n = 0; n < mm; ++n) {
                const float hi = tf32_rna_host(k[n]);
                const float lo = tf32_rna_host(k[n] - hi);
                float* dst = h.data() + (size_t)t * per_stage + (size_t)s8 * 2 * 2 * nb * 4;
                dst[((0 * 2 + c2) * nb + n) * 4 + e] = hi;
                dst[((1 * 2 + c2) * nb + n) * 4 + e] = lo;
            }
        }
    float* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, h.size() * sizeof(float)));
    CUDA_TRY(cudaMemcpy(d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
    md->d_aop = d;
    md->aop_stage = per_stage;
    return TNRD_OK;
}

// One stage as phi_kernel + adj_kernel.  Returns -1 when this model / launch
// is not supported (the caller falls back to the CUDA-core kernels).
template <int MS>
static int launch_adj_m(const tnrd_model* md, const StageArgs& a, int batch, cudaStream_t s) {
    using K = StageKernel<MS, true, LargeTile>;
    using AC = adj::AdjCfg<MS>;
    constexpr int RF = 4, TM = K::kTmTile, R = MS / 2;
    using PC = adj::PhiCfg<MS, RF>;
    if constexpr (!K::kPT) return -1;
    if (!md->fast || !a.tab3 || !K::pt_fits(a)) return -1;
    if (a.flags & (TNRD_STAGE_TOP_HALO | TNRD_STAGE_BOTTOM_HALO)) return -1;   // strips: CUDA-core kernels
    const int pairs = (md->nk + 1) / 2;
    const int kc = round_up((pairs + 1) / 2, 2);           // 4-filter chunks, whole K-steps of 8
    const size_t adj_smem = AC::smem_bytes(kc);
    if (adj_smem > 227 * 1024) return -1;
    int rc = adj_operand(md, AC::NB, kc);
    if (rc) return rc;
    const int G = (a.W + AC::GW - 1) / AC::GW;
    adj::AdjArgs q;
    q.kc = kc;
    q.xp = G * AC::GW + 2 * R;
    q.phi_row = (int64_t)kc * q.xp * 4;
    q.phi_img = (int64_t)(a.H + 2 * R) * q.phi_row;
    q.bop = md->d_aop + (size_t)a.stage * md->aop_stage;
    q.rows_per_cta = std::min(a.H, 128);
    // phi workspace of this stream: as many images per pass as fit the budget
    static const size_t budget = [] {
        const char* e = std::getenv("TNRD_ADJ_WS_MB");
        const long mb = e ? std::atol(e) : 4096;
        return (size_t)std::max(64L, mb) << 20;
    }();
    const size_t img_bytes = (size_t)q.phi_img * sizeof(float);
    if (img_bytes > budget) return -1;   // one image's phi must fit the workspace (a 16384^2 scene: 52 GB)
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)batch, budget / img_bytes));
    const std::vector<long> key = {a.H, a.W, kc, MS};
    float* phi = nullptr;
    {
        std::lock_guard<std::mutex> lk(md->ws_mu);
        auto& b = md->aws[s];
        const size_t bytes = (size_t)chunk * img_bytes;
        if (b.bytes < bytes || b.key != key) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            CUDA_TRY(cudaStreamIsCapturing(s, &cs));
            if (cs != cudaStreamCaptureStatusNone)
                return fail(TNRD_ECUDA, "adjoint workspace must be allocated before stream capture");
            if (b.bytes < bytes) {
                if (b.ptr) md->retired.push_back(b.ptr);   // a captured graph may still use it
                b.ptr = nullptr;
                CUDA_TRY(cudaMalloc(&b.ptr, bytes));
                b.bytes = bytes;
            }
            // cells no kernel writes (padding columns, all-zero filter chunks) must be finite
            CUDA_TRY(cudaMemsetAsync(b.ptr, 0, b.bytes, s));
            b.key = key;
        }
        phi = static_cast<float*>(b.ptr);
    }
    q.phi = phi;
    using TB = typename K::TB;
    auto pk = adj::phi_kernel<MS, RF, TM, TB>;
    auto ak = adj::adj_kernel<MS>;
    static std::mutex mu;
    static uint64_t attr_set = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!(attr_set & (1ull << (dev & 63)))) {
            CUDA_TRY(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
            CUDA_TRY(cudaFuncSetAttribute(ak, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            attr_set |= 1ull << (dev & 63);
        }
    }
    TB tb;
    const float* htaps = md->h_taps.data() + (size_t)a.stage * md->nk_pad * md->kp;
    K::template fill_taps<TM, 2>(tb, htaps, a.nk);
    const size_t phi_smem = PC::smem_bytes(a.tab3_stride);
    for (int b0 = 0; b0 < batch; b0 += chunk) {
        const int nb = std::min(chunk, batch - b0);
        StageArgs c = a;
        c.ngroups = pairs;
        c.u_in = a.u_in + (int64_t)b0 * a.img_stride;
        c.f = a.f + (int64_t)b0 * a.img_stride;
        c.u_out = a.u_out + (int64_t)b0 * a.img_stride;
        if (a.force_out) c.force_out = a.force_out + (int64_t)b0 * a.img_stride;
        const dim3 pg((a.W + adj::kPhiTile - 1) / adj::kPhiTile, (a.H + adj::kPhiTile - 1) / adj::kPhiTile, nb);
        pk<<<pg, adj::kPhiThreads, phi_smem, s>>>(c, q, tb);
        CUDA_TRY(cudaGetLastError());
        const dim3 ag(G, (a.H + q.rows_per_cta - 1) / q.rows_per_cta, nb);
        ak<<<ag, adj::kAdjThreads, adj_smem, s>>>(c, q);
        CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(2);
    }
    return TNRD_OK;
}

static int launch_adj(const tnrd_model* md, const StageArgs& a, int batch, cudaStream_t s) {
    switch (md->m) {
        case 5: return launch_adj_m<5>(md, a, batch, s);
        case 7: return launch_adj_m<7>(md, a, batch, s);
        default: return -1;
    }
}

static int launch_stage(const tnrd_model* md, int t, const float* u_in, const float* f,
                        float* u_out, int batch, int H, int W, int64_t ld, int64_t image_stride,
                        uint32_t flags, uint32_t* d_status, cudaStream_t s, float* force_out = nullptr) {
    StageArgs a = stage_args(md, t, flags);
    a.u_in = u_in; a.f = f; a.u_out = u_out;
    a.force_out = force_out;
    a.ld = ld; a.img_stride = image_stride;
    a.H = H; a.W = W;
    a.status = d_status;
    const int mode = g_kernel_mode.load();
#ifdef TNRD_EXPERIMENTS
    if (mode == 2 && tc3_supported(md)) return dispatch_tc3(md, t, a, batch, s);
    if (mode == 5 && tc_supported(md)) return dispatch_tc(md, t, a, batch, s);
    if (mode == 8 && zf_supported(md)) return launch_zf(md, t, a, batch, s);
#endif
    if (mode == 2 || mode == 5 || mode == 8)
        return fail(TNRD_EUNSUPPORTED, "tensor-core stage kernel unavailable for this model");
    if (mode == 12) {
        const int rc = launch_adj(md, a, batch, s);
        if (rc != -1) return rc;   // ran (or failed); -1: unsupported here, CUDA-core kernels
    }
    return md->fast ? dispatch_m<true>(md, a, batch, s) : dispatch_m<false>(md, a, batch, s);
}

extern "C" int tnrd_stage(const tnrd_model* md, int t, const float* u_in, const float* f,
                          float* u_out, int batch, int H, int W, int64_t ld, int64_t image_stride,
                          uint32_t flags, uint32_t* d_status, void* stream) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (t < 0 || t >= md->T) return fail(TNRD_EINVAL, "stage %d out of range [0, %d)", t, md->T);
    if (!u_in || !f || !u_out || !d_status) return fail(TNRD_EINVAL, "NULL buffer");
    if (u_in == u_out) return fail(TNRD_EINVAL, "u_in and u_out must not alias");
    int rc = check_shape(md, batch, H, W, ld, image_stride);
    if (rc) return rc;
    DeviceGuard dg(md->device);
    return launch_stage(md, t, u_in, f, u_out, batch, H, W, ld, image_stride, flags, d_status,
                        (cudaStream_t)stream);
}

// diffusion_step with its force (diffusion.py:184-194 returns u_next and,
// through the trace, u~ = u - force): both outputs from one launch.
extern "C" int tnrd_stage_force(const tnrd_model* md, int t, const float* u_in, const float* f,
                                float* u_out, float* force_out, int batch, int H, int W, int64_t ld,
                                int64_t image_stride, uint32_t flags, uint32_t* d_status, void* stream) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (t < 0 || t >= md->T) return fail(TNRD_EINVAL, "stage %d out of range [0, %d)", t, md->T);
    if (!u_in || !f || !u_out || !force_out || !d_status) return fail(TNRD_EINVAL, "NULL buffer");
    if (u_in == u_out || force_out == u_out || force_out == u_in)
        return fail(TNRD_EINVAL, "u_in, u_out and force_out must not alias");
    if (flags & TNRD_STAGE_FORCE) return fail(TNRD_EINVAL, "TNRD_STAGE_FORCE makes u_out the force already");
    int rc = check_shape(md, batch, H, W, ld, image_stride);
    if (rc) return rc;
    if (g_kernel_mode.load() == 2 || g_kernel_mode.load() == 5 || g_kernel_mode.load() == 8)
        return fail(TNRD_EUNSUPPORTED, "tnrd_stage_force runs the CUDA-core stage kernels only");
    DeviceGuard dg(md->device);
    return launch_stage(md, t, u_in, f, u_out, batch, H, W, ld, image_stride, flags, d_status,
                        (cudaStream_t)stream, force_out);
}

#ifdef TNRD_EXPERIMENTS
// One fused dataflow launch for all T stages (mode 9).  Returns -1 when not
// applicable.
template <bool FAST>
static int despeckle_fused_m(const tnrd_model* md, const StageArgs* st, int batch, cudaStream_t s) {
    switch (md->m) {
        case 3: return StageKernel<3, FAST, SplitTile>::launch_fused(md, st, md->T, batch, s);
        case 5: return StageKernel<5, FAST, SplitTile>::launch_fused(md, st, md->T, batch, s);
        case 7: return StageKernel<7, FAST, SplitTile>::launch_fused(md, st, md->T, batch, s);
        default: return StageKernel<9, FAST, SplitTile>::launch_fused(md, st, md->T, batch, s);
    }
}

static int despeckle_fused(const tnrd_model* md, const float* f, float* u_out, float* work, int batch,
                           int H, int W, int64_t ld, int64_t image_stride, uint32_t* d_status,
                           cudaStream_t s) {
    // opt-in (mode 9): measured slower than the per-stage split kernel on
    // C2, kept for the dataflow experiments
    const int mode = g_kernel_mode.load();
    if (mode != 9) return -1;
    if (md->T > kMaxFusedStages || md->T < 1) return -1;
    StageArgs st[kMaxFusedStages];
    const float* cur = f;
    for (int t = 0; t < md->T; ++t) {
        float* dst = ((md->T - 1 - t) % 2 == 0) ? u_out : work;
        const uint32_t fl = t == 0 ? (TNRD_STAGE_FLOOR_INPUT | TNRD_STAGE_CHECK_F) : 0u;
        st[t] = stage_args(md, t, fl);
        st[t].u_in = cur; st[t].f = f; st[t].u_out = dst;
        st[t].ld = ld; st[t].img_stride = image_stride;
        st[t].H = H; st[t].W = W;
        st[t].status = d_status;
        cur = dst;
    }
    const int ng = (md->nk + SplitTile::F - 1) / SplitTile::F;
    const long tiles = StageKernel<7, true, SplitTile>::tiles(st[0], batch);
    if (ng > 63 || tiles >= (1l << 18)) return -1;
    if ((size_t)tiles * ng * SplitTile::TH * SplitTile::TW * sizeof(float) * 2 > kMaxSplitBytes) return -1;
    return md->fast ? despeckle_fused_m<true>(md, st, batch, s) : despeckle_fused_m<false>(md, st, batch, s);
}

#else
static int despeckle_fused(const tnrd_model* md, const float*, float*, float*, int, int, int, int64_t,
                           int64_t, uint32_t*, cudaStream_t) {
    (void)md;
    if (g_kernel_mode.load() == 9) return fail(TNRD_EUNSUPPORTED, "fused dataflow kernel not built (TNRD_EXPERIMENTS)");
    return -1;
}
#endif  // TNRD_EXPERIMENTS

static int despeckle_stages(const tnrd_model* md, const float* f, float* u_out, float* work,
                            int batch, int H, int W, int64_t ld, int64_t image_stride,
                            uint32_t* d_status, cudaStream_t s) {
    const float* cur = f;
    for (int t = 0; t < md->T; ++t) {
        float* dst = ((md->T - 1 - t) % 2 == 0) ? u_out : work;
        const uint32_t fl = t == 0 ? (TNRD_STAGE_FLOOR_INPUT | TNRD_STAGE_CHECK_F) : 0u;
        int rc = launch_stage(md, t, cur, f, dst, batch, H, W, ld, image_stride, fl, d_status, s);
        if (rc) return rc;
        cur = dst;
    }
    return TNRD_OK;
}

// Batch fork (DESIGN.md §7b item 5, measured with tools/multistream_probe.py):
// in auto mode, when even the smaller half of the batch selects the
// large-tile kernel (>= 3 waves), run the halves on two streams.  Returns the
// fork resources of caller stream s, or nullptr for one stream.
// TNRD_BATCH_FORK=0 turns it off (A/B runs).
static const tnrd_model::ForkRes* batch_fork(const tnrd_model* md, int batch, int H, int W,
                                             cudaStream_t s) {
    static const bool enabled = [] {
        const char* e = std::getenv("TNRD_BATCH_FORK");
        return !(e && e[0] == '0');
    }();
    if (!enabled || batch < 2 || g_kernel_mode.load() != 0) return nullptr;
    // the fork resources are keyed by the caller's stream handle: the
    // per-thread default stream is a different stream in every thread under
    // one handle, so it never forks
    if (s == cudaStreamPerThread) return nullptr;
    StageArgs a = stage_args(md, 0, 0u);
    a.H = H; a.W = W;
    if (!use_large_tiles(a, batch / 2)) return nullptr;   // each half >= 3 waves of the tile kernel
    std::lock_guard<std::mutex> lk(md->ws_mu);
    auto& fr = md->forks[s];
    if (!fr.s2) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
            return nullptr;   // resources are created outside any capture
        int prio = 0;
        cudaStreamGetPriority(s, &prio);
        if (cudaStreamCreateWithPriority(&fr.s2, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&fr.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&fr.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            if (fr.s2) cudaStreamDestroy(fr.s2);
            if (fr.fork) cudaEventDestroy(fr.fork);
            md->forks.erase(s);
            return nullptr;
        }
    }
    return &fr;
}

extern "C" int tnrd_despeckle(const tnrd_model* md, const float* f, float* u_out, float* work,
                              int batch, int H, int W, int64_t ld, int64_t image_stride,
                              uint32_t* d_status, void* stream) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (!f || !u_out || !d_status || (md->T > 1 && !work)) return fail(TNRD_EINVAL, "NULL buffer");
    if (f == u_out || f == work || u_out == work) return fail(TNRD_EINVAL, "buffers must not alias");
    int rc = check_shape(md, batch, H, W, ld, image_stride);
    if (rc) return rc;
    DeviceGuard dg(md->device);
    cudaStream_t s = (cudaStream_t)stream;
    rc = despeckle_fused(md, f, u_out, work, batch, H, W, ld, image_stride, d_status, s);
    if (rc != -1) return rc;   // ran (or failed) as one fused launch
    const tnrd_model::ForkRes* fr = batch_fork(md, batch, H, W, s);
    if (!fr) return despeckle_stages(md, f, u_out, work, batch, H, W, ld, image_stride, d_status, s);
    // images are independent: the two halves' stage chains run on two
    // streams, so one half's stage t + 1 fills the SMs the other's last tile
    // wave of stage t leaves idle.  Same kernel for both halves and the
    // whole batch, so the same bits.  Capture-safe (event fork / join).
    const int b0 = (batch + 1) / 2;
    const int64_t off = (int64_t)b0 * image_stride;
    VariantGuard vg(1);   // both halves on the large-tile kernel
    CUDA_TRY(cudaEventRecord(fr->fork, s));
    CUDA_TRY(cudaStreamWaitEvent(fr->s2, fr->fork, 0));
    rc = despeckle_stages(md, f, u_out, work, b0, H, W, ld, image_stride, d_status, s);
    if (rc == TNRD_OK)
        rc = despeckle_stages(md, f + off, u_out + off, work ? work + off : nullptr, batch - b0, H, W,
                              ld, image_stride, d_status, fr->s2);
    // join even after a failed launch, so a capture on s stays well formed
    CUDA_TRY(cudaEventRecord(fr->join, fr->s2));
    CUDA_TRY(cudaStreamWaitEvent(s, fr->join, 0));
    return rc;
}

// ----------------------------------------------------------------- plans

struct tnrd_plan {
    const tnrd_model* md = nullptr;
    int batch = 0, H = 0, W = 0;
    cudaStream_t stream = nullptr;
    float *d_f = nullptr, *d_u = nullptr, *d_work = nullptr;
    uint32_t* d_status = nullptr;
    uint32_t* h_status = nullptr;  // pinned
    // the T stage launches on the plan's own buffers, captured once as a CUDA
    // graph (status reset + T kernels) and replayed: one launch per call
    cudaGraphExec_t graph = nullptr;
    int graph_mode = -1;           // stage-kernel mode the graph was captured with
    uint64_t graph_launches = 0;   // kernels in the graph
    long runs = 0;
    // streaming (tnrd_plan_despeckle_host_many): chained twin plans, each on
    // its own stream, take images round-robin so copies and stages overlap
    tnrd_plan* twin = nullptr;
    uint32_t* h_status_many = nullptr;  // pinned, 2 words per image
    int h_status_cap = 0;
    // banded host path for one large scene (plan_banded_host): row bands on
    // their own streams, H2D / D2H streams, per-band events
    int nbands = 0;
    std::vector<cudaStream_t> band_streams;
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_stage;  // [band], [2][band]
    cudaEvent_t ev_reset = nullptr;
};

extern "C" int tnrd_plan_destroy(tnrd_plan* p) {
    if (!p) return TNRD_OK;
    {
        DeviceGuard dg(p->md->device);
        if (p->stream) cudaStreamSynchronize(p->stream);
        if (p->graph) cudaGraphExecDestroy(p->graph);
        cudaFree(p->d_f); cudaFree(p->d_u); cudaFree(p->d_work); cudaFree(p->d_status);
        if (p->h_status) cudaFreeHost(p->h_status);
        if (p->h_status_many) cudaFreeHost(p->h_status_many);
        for (cudaStream_t bs : p->band_streams) { cudaStreamSynchronize(bs); cudaStreamDestroy(bs); }
        if (p->copy_in) { cudaStreamSynchronize(p->copy_in); cudaStreamDestroy(p->copy_in); }
        if (p->copy_out) { cudaStreamSynchronize(p->copy_out); cudaStreamDestroy(p->copy_out); }
        for (cudaEvent_t e : p->ev_in) cudaEventDestroy(e);
        for (cudaEvent_t e : p->ev_stage) cudaEventDestroy(e);
        if (p->ev_reset) cudaEventDestroy(p->ev_reset);
        if (p->stream) cudaStreamDestroy(p->stream);
    }
    tnrd_plan* twin = p->twin;
    delete p;
    if (twin) tnrd_plan_destroy(twin);
    return TNRD_OK;
}

extern "C" int tnrd_plan_create(const tnrd_model* md, int batch, int H, int W, tnrd_plan** out) {
    if (!out) return fail(TNRD_EINVAL, "out is NULL");
    *out = nullptr;
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    int rc = check_shape(md, batch, H, W, W, (int64_t)W * H);
    if (rc) return rc;
    DeviceGuard dg(md->device);
    auto* p = new tnrd_plan();
    p->md = md; p->batch = batch; p->H = H; p->W = W;
    const size_t n = (size_t)batch * H * W;
    cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_f, n * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_u, n * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_work, n * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_status, TNRD_STATUS_WORDS * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMallocHost(&p->h_status, TNRD_STATUS_WORDS * sizeof(uint32_t));
    if (e != cudaSuccess) {
        tnrd_plan_destroy(p);
        return fail(TNRD_ECUDA, "plan allocation failed: %s", cudaGetErrorString(e));
    }
    *out = p;
    return TNRD_OK;
}

static int plan_eager(tnrd_plan* p, const float* f_dev, float* u_dev) {
    int rc = tnrd_status_reset(p->d_status, p->stream);
    if (rc) return rc;
    return tnrd_despeckle(p->md, f_dev, u_dev, p->d_work, p->batch, p->H, p->W, p->W,
                          (int64_t)p->W * p->H, p->d_status, p->stream);
}

static int plan_run(tnrd_plan* p, const float* f_dev, float* u_dev) {
    const bool own = f_dev == p->d_f && u_dev == p->d_u;
    const int mode = g_kernel_mode.load();
    // first call eager (sets kernel attributes outside any capture); later
    // calls on the plan's own buffers replay a captured graph
    if (!own || p->runs++ == 0) return plan_eager(p, f_dev, u_dev);
    if (!p->graph || p->graph_mode != mode) {
        if (p->graph) { cudaGraphExecDestroy(p->graph); p->graph = nullptr; }
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
            return plan_eager(p, f_dev, u_dev);
        const uint64_t before = g_launches.load();
        int rc = plan_eager(p, f_dev, u_dev);
        cudaError_t e = cudaStreamEndCapture(p->stream, &g);
        const uint64_t captured = g_launches.load() - before;
        g_launches.store(before);  // captured, not launched
        if (rc) {
            // e.g. a workspace that must grow first: run eagerly this time
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return plan_eager(p, f_dev, u_dev);
        }
        if (e != cudaSuccess || cudaGraphInstantiate(&p->graph, g, 0) != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            p->graph = nullptr;
            return plan_eager(p, f_dev, u_dev);
        }
        cudaGraphDestroy(g);
        p->graph_mode = mode;
        p->graph_launches = captured;
    }
    CUDA_TRY(cudaGraphLaunch(p->graph, p->stream));
    g_launches.fetch_add(p->graph_launches);
    return TNRD_OK;
}

extern "C" int tnrd_plan_despeckle_device(tnrd_plan* p, const float* f_dev, float* u_dev) {
    if (!p) return fail(TNRD_EINVAL, "plan is NULL");
    DeviceGuard dg(p->md->device);
    return plan_run(p, f_dev ? f_dev : p->d_f, u_dev ? u_dev : p->d_u);
}

extern "C" int tnrd_plan_check(tnrd_plan* p, int* bad_stage) {
    if (!p) return fail(TNRD_EINVAL, "plan is NULL");
    DeviceGuard dg(p->md->device);
    CUDA_TRY(cudaMemcpyAsync(p->h_status, p->d_status, TNRD_STATUS_WORDS * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return tnrd_status_decode(p->h_status, bad_stage);
}

// Row bands for one large scene: band boundaries on multiples of the large
// tile height (the band launches then see the same tile grid as the whole
// image, so the result is bit-identical), every band >= 3 waves of large
// tiles (the tile kernel, as for the whole image), at most 16 bands.
// 0 = do not band (small images, batches, CUDA-core kernels not in auto mode).
static int band_count(const tnrd_model* md, int batch, int H, int W) {
    static const int env = [] {
        const char* e = getenv("TNRD_SCENE_BANDS");
        return e ? std::min(std::max(atoi(e), 1), 64) : 0;
    }();
    if (batch != 1 || g_kernel_mode.load() != 0) return 0;
    const long tiles_x = (W + LargeTile::TW - 1) / LargeTile::TW;
    const long row_tiles = (H + LargeTile::TH - 1) / LargeTile::TH;
    const long wave3 = 3L * 2 * sm_count();
    // the whole scene must select the tile kernel in auto mode (cc_variant)
    if (row_tiles * tiles_x < 2 * wave3) return 0;
    long nb = env ? env : std::min<long>(16, (row_tiles * tiles_x) / wave3);
    nb = std::min(nb, row_tiles);
    return nb >= 2 ? (int)nb : 0;
}

static int banded_setup(tnrd_plan* p, int nb) {
    if (p->nbands == nb) return TNRD_OK;
    for (cudaStream_t bs : p->band_streams) { cudaStreamSynchronize(bs); cudaStreamDestroy(bs); }
    for (cudaEvent_t e : p->ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_stage) cudaEventDestroy(e);
    p->band_streams.clear(); p->ev_in.clear(); p->ev_stage.clear();
    p->nbands = 0;
    if (!p->copy_in) CUDA_TRY(cudaStreamCreateWithFlags(&p->copy_in, cudaStreamNonBlocking));
    if (!p->copy_out) CUDA_TRY(cudaStreamCreateWithFlags(&p->copy_out, cudaStreamNonBlocking));
    if (!p->ev_reset) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_reset, cudaEventDisableTiming));
    p->band_streams.resize(nb);
    p->ev_in.resize(nb);
    p->ev_stage.resize(2 * (size_t)nb);
    for (int b = 0; b < nb; ++b) {
        CUDA_TRY(cudaStreamCreateWithFlags(&p->band_streams[b], cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_in[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_stage[b], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->ev_stage[nb + b], cudaEventDisableTiming));
    }
    p->nbands = nb;
    return TNRD_OK;
}

// One large scene from/to HOST memory with the copies overlapped: the scene
// is cut into nb row bands; band b's H2D, its T stage launches (row-strip
// halo mode: the neighbouring bands' rows are read in place) and its D2H
// run on their own streams, ordered by events only where the data flows --
// stage t of band b after stage t-1 of bands b-1, b, b+1 (its halo rows;
// also the write-after-read of the ping-pong buffer), stage 0 after the
// H2D of bands b-1..b+1, the D2H of band b after its last stage.  So the
// first stages start after 2/nb of the input has landed and the last
// bands' output copies overlap the remaining stages.
static int plan_banded_host(tnrd_plan* p, const float* f_host, float* u_host, int nb) {
    const tnrd_model* md = p->md;
    int rc = banded_setup(p, nb);
    if (rc) return rc;
    VariantGuard vg(1);   // every band on the whole scene's kernel (large tiles)
    // work queued earlier on the plan's stream (tnrd_plan_despeckle_device
    // returns without a sync) uses the same buffers: the copy and band
    // streams start after it
    CUDA_TRY(cudaEventRecord(p->ev_reset, p->stream));
    CUDA_TRY(cudaStreamWaitEvent(p->copy_in, p->ev_reset, 0));
    for (cudaStream_t bs : p->band_streams) CUDA_TRY(cudaStreamWaitEvent(bs, p->ev_reset, 0));
    const int H = p->H, W = p->W, T = md->T;
    const int row_tiles = (H + LargeTile::TH - 1) / LargeTile::TH;
    std::vector<int> r0(nb + 1);
    for (int b = 0; b <= nb; ++b) r0[b] = std::min(H, (int)((long)row_tiles * b / nb) * LargeTile::TH);
    rc = tnrd_status_reset(p->d_status, p->copy_in);
    if (rc) return rc;
    for (int b = 0; b < nb; ++b) {
        const size_t off = (size_t)r0[b] * W, n = (size_t)(r0[b + 1] - r0[b]) * W;
        CUDA_TRY(cudaMemcpyAsync(p->d_f + off, f_host + off, n * sizeof(float), cudaMemcpyHostToDevice,
                                 p->copy_in));
        CUDA_TRY(cudaEventRecord(p->ev_in[b], p->copy_in));
    }
    for (int t = 0; t < T; ++t) {
        const float* src = t == 0 ? p->d_f : (((T - t) % 2 == 0) ? p->d_u : p->d_work);
        float* dst = ((T - 1 - t) % 2 == 0) ? p->d_u : p->d_work;
        cudaEvent_t* prev = p->ev_stage.data() + (size_t)((t + 1) % 2) * nb;
        cudaEvent_t* cur = p->ev_stage.data() + (size_t)(t % 2) * nb;
        for (int b = 0; b < nb; ++b) {
            cudaStream_t s = p->band_streams[b];
            for (int nbh = std::max(0, b - 1); nbh <= std::min(nb - 1, b + 1); ++nbh) {
                if (t == 0) CUDA_TRY(cudaStreamWaitEvent(s, p->ev_in[nbh], 0));
                else if (nbh != b) CUDA_TRY(cudaStreamWaitEvent(s, prev[nbh], 0));
            }
            uint32_t fl = t == 0 ? (TNRD_STAGE_FLOOR_INPUT | TNRD_STAGE_CHECK_F) : 0u;
            if (b > 0) fl |= TNRD_STAGE_TOP_HALO;
            if (b + 1 < nb) fl |= TNRD_STAGE_BOTTOM_HALO;
            const size_t off = (size_t)r0[b] * W;
            rc = launch_stage(md, t, src + off, p->d_f + off, dst + off, 1, r0[b + 1] - r0[b], W, W,
                              (int64_t)W * H, fl, p->d_status, s);
            if (rc) return rc;
            CUDA_TRY(cudaEventRecord(cur[b], s));
        }
    }
    cudaEvent_t* last = p->ev_stage.data() + (size_t)((T - 1) % 2) * nb;
    for (int b = 0; b < nb; ++b) {
        const size_t off = (size_t)r0[b] * W, n = (size_t)(r0[b + 1] - r0[b]) * W;
        CUDA_TRY(cudaStreamWaitEvent(p->copy_out, last[b], 0));
        CUDA_TRY(cudaMemcpyAsync(u_host + off, p->d_u + off, n * sizeof(float), cudaMemcpyDeviceToHost,
                                 p->copy_out));
    }
    CUDA_TRY(cudaMemcpyAsync(p->h_status, p->d_status, TNRD_STATUS_WORDS * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, p->copy_out));
    CUDA_TRY(cudaStreamSynchronize(p->copy_out));
    int bad = -1;
    return tnrd_status_decode(p->h_status, &bad);
}

extern "C" int tnrd_plan_despeckle_host(tnrd_plan* p, const float* f_host, float* u_host) {
    if (!p) return fail(TNRD_EINVAL, "plan is NULL");
    if (!f_host || !u_host) return fail(TNRD_EINVAL, "NULL host buffer");
    DeviceGuard dg(p->md->device);
    const int nb = band_count(p->md, p->batch, p->H, p->W);
    if (nb >= 2) return plan_banded_host(p, f_host, u_host, nb);
    const size_t bytes = (size_t)p->batch * p->H * p->W * sizeof(float);
    CUDA_TRY(cudaMemcpyAsync(p->d_f, f_host, bytes, cudaMemcpyHostToDevice, p->stream));
    int rc = plan_run(p, p->d_f, p->d_u);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(u_host, p->d_u, bytes, cudaMemcpyDeviceToHost, p->stream));
    int bad = -1;
    return tnrd_plan_check(p, &bad);
}

// A sequence of `count` host images (each batch*H*W fp32, dense, back to
// back): image i's H2D, T stages and D2H are issued round-robin on the plan
// and its chained twins (own streams and buffers), so the copies of one
// image overlap the stages of the next and small images run concurrently.  Host buffers should be pinned for the overlap (pageable ones work,
// serialised).  Returns the first image's error, with *bad_index set (-1 if
// none).
extern "C" int tnrd_plan_despeckle_host_many(tnrd_plan* p, const float* f_host, float* u_host,
                                             int count, int* bad_index) {
    if (bad_index) *bad_index = -1;
    if (!p) return fail(TNRD_EINVAL, "plan is NULL");
    if (count < 0) return fail(TNRD_EINVAL, "count must be >= 0");
    if (count == 0) return TNRD_OK;
    if (!f_host || !u_host) return fail(TNRD_EINVAL, "NULL host buffer");
    DeviceGuard dg(p->md->device);
    // pipeline depth: the plan plus depth-1 chained twins, each on its own
    // stream, take the images round-robin.  Measured on B200 (C2 e2e,
    // MPix/s): depth 1 476, 2 568, 3 600, 4 616 (r01 split kernels); with
    // the r01 cubic kernels 4 726, 6 763, 8 764.  A batch that fills the GPU
    // by itself gains nothing (C5: 174 / 178 / 179), so deep pipelines are
    // kept to plans of <= 64 MB per buffer.
    static const int depth_env = [] {
        const char* e = getenv("TNRD_STREAM_DEPTH");
        return e ? std::min(std::max(atoi(e), 1), 8) : 0;
    }();
    const size_t plan_bytes = (size_t)p->batch * p->H * p->W * sizeof(float);
    const int depth = depth_env ? depth_env : (plan_bytes <= (size_t(64) << 20) ? 6 : 2);
    std::vector<tnrd_plan*> ring{p};
    for (int d = 1; d < depth; ++d) {
        tnrd_plan* last = ring.back();
        if (!last->twin) {
            int rc = tnrd_plan_create(p->md, p->batch, p->H, p->W, &last->twin);
            if (rc) return rc;
        }
        ring.push_back(last->twin);
    }
    if (p->h_status_cap < count) {
        if (p->h_status_many) cudaFreeHost(p->h_status_many);
        p->h_status_many = nullptr;
        p->h_status_cap = 0;
        CUDA_TRY(cudaMallocHost(&p->h_status_many, (size_t)count * TNRD_STATUS_WORDS * sizeof(uint32_t)));
        p->h_status_cap = count;
    }
    const size_t n = (size_t)p->batch * p->H * p->W;
    for (int i = 0; i < count; ++i) {
        tnrd_plan* q = ring[i % ring.size()];
        CUDA_TRY(cudaMemcpyAsync(q->d_f, f_host + i * n, n * sizeof(float), cudaMemcpyHostToDevice,
                                 q->stream));
        int rc = plan_run(q, q->d_f, q->d_u);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(u_host + i * n, q->d_u, n * sizeof(float), cudaMemcpyDeviceToHost,
                                 q->stream));
        CUDA_TRY(cudaMemcpyAsync(p->h_status_many + (size_t)i * TNRD_STATUS_WORDS, q->d_status,
                                 TNRD_STATUS_WORDS * sizeof(uint32_t), cudaMemcpyDeviceToHost, q->stream));
    }
    for (tnrd_plan* q : ring) CUDA_TRY(cudaStreamSynchronize(q->stream));
    for (int i = 0; i < count; ++i) {
        int bad = -1;
        const int rc = tnrd_status_decode(p->h_status_many + (size_t)i * TNRD_STATUS_WORDS, &bad);
        if (rc) {
            if (bad_index) *bad_index = i;
            return rc;
        }
    }
    return TNRD_OK;
}

extern "C" void* tnrd_plan_stream(tnrd_plan* p) { return p ? (void*)p->stream : nullptr; }
extern "C" float* tnrd_plan_f_device(tnrd_plan* p) { return p ? p->d_f : nullptr; }
extern "C" float* tnrd_plan_u_device(tnrd_plan* p) { return p ? p->d_u : nullptr; }

#ifdef TNRD_FUSED_TRACE
extern "C" __attribute__((visibility("default"))) int tnrd_debug_fused_trace(long long* out, int n) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out, fused::g_fused_trace, (size_t)std::min(n, 4096) * 5 * sizeof(long long)));
    return TNRD_OK;
}
#endif

#ifdef TNRD_SPLIT_TRACE
extern "C" __attribute__((visibility("default"))) int tnrd_debug_split_trace(unsigned long long* out, int n) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out, g_split_trace, (size_t)std::min(n, 4096) * 4 * sizeof(unsigned long long)));
    return TNRD_OK;
}
#endif

// ----------------------------------------------------------------- training backward

// stream-ordered scratch freed on scope exit (after the caller's sync)
struct StreamScratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit StreamScratch(cudaStream_t st) : s(st) {}
    template <class T>
    cudaError_t get(T** p, size_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(count, 1) * sizeof(T), s);
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = static_cast<T*>(q);
        return e;
    }
    ~StreamScratch() {
        for (void* q : ptrs) cudaFreeAsync(q, s);
    }
};

// the image-space backward kernels of one filter chunk, each as an interior
// launch and a border-band launch
template <int MS>
static void bwd_image_kernels(const tnrd_model* md, const train::BwdArgs& a, int H, int W, bool gprev,
                              cudaStream_t s) {
    for (int pass = 0; pass < 3; ++pass) {
        if (pass == 2 && !gprev) break;
        for (int part_i = 0; part_i < 2; ++part_i) {
            const train::PixelSet ps = train::pixel_set(H, W, MS / 2, part_i == 0);
            if (ps.n == 0) continue;
            const dim3 grid((unsigned)((ps.n + 255) / 256), (unsigned)a.nf);
            if (pass == 0) {
                if (md->fast) train::bwd_maps_kernel<MS, true><<<grid, 256, 0, s>>>(a, ps);
                else train::bwd_maps_kernel<MS, false><<<grid, 256, 0, s>>>(a, ps);
            } else if (pass == 1) {
                train::bwd_v_kernel<MS><<<grid, 256, 0, s>>>(a, ps);
            } else {
                train::bwd_adj_kernel<MS><<<grid, 256, 0, s>>>(a, ps);
            }
            g_launches.fetch_add(1);
        }
    }
    if (gprev) {
        train::bwd_gprev_kernel<<<(unsigned)((H * W + 255) / 256), 256, 0, s>>>(a);
        g_launches.fetch_add(1);
    }
}

// training.py:69-123 (_stage_backward) for one dense H x W image on the GPU
// (tnrd_train.cuh).  Device inputs u_prev, f, g_next (NULL = zero adjoint);
// g_prev: device output (NULL: not wanted).  Host outputs (NULL: not
// wanted): *grad_beta, grad_k[nk][m*m] (the kernel-space gradient gk_i of
// training.py:108-110, before the basis map), grad_w[nk][M].  Synchronous.
extern "C" int tnrd_stage_backward(const tnrd_model* md, int t, const float* u_prev, const float* f,
                                   const float* g_next, float* g_prev, int H, int W,
                                   double* grad_beta, double* grad_k, double* grad_w, void* stream) {
    if (!md) return fail(TNRD_EINVAL, "model is NULL");
    if (t < 0 || t >= md->T) return fail(TNRD_EINVAL, "stage %d out of range [0, %d)", t, md->T);
    if (!u_prev || !f) return fail(TNRD_EINVAL, "NULL buffer");
    int rc = check_shape(md, 1, H, W, W, (int64_t)W * H);
    if (rc) return rc;
    DeviceGuard dg(md->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int n = H * W;
    const int m = md->m, mm = m * m, M = md->M, nk = md->nk;
    const int nout = 2 * mm + M;
    const int nfc = std::min(nk, 16);
    const int nseg = (W + train::kSeg - 1) / train::kSeg;
    const int nblk = H * nseg;                 // bwd_reduce_kernel blocks per filter
    const bool want_params = grad_beta || grad_k || grad_w;
    StreamScratch scr(s);
    float *force, *g_t, *z, *phi, *dphi, *v, *w1, *adjb, *gp;
    double *part, *outd;
    uint32_t* status;
    const size_t maps = (size_t)nfc * n;
    if (scr.get(&force, n) || scr.get(&g_t, n) || scr.get(&z, maps) || scr.get(&phi, maps) ||
        scr.get(&dphi, maps) || scr.get(&v, maps) || scr.get(&w1, maps) ||
        (g_prev && scr.get(&adjb, maps)) || scr.get(&gp, n) ||
        scr.get(&part, std::max<size_t>((size_t)nfc * nblk * nout, (size_t)(n + 255) / 256)) ||
        scr.get(&outd, (size_t)nfc * nout) || scr.get(&status, TNRD_STATUS_WORDS))
        return fail(TNRD_ECUDA, "backward workspace allocation failed");
    rc = tnrd_status_reset(status, s);
    if (rc) return rc;
    // force(u_prev) by the fused stage kernel (TNRD_STAGE_FORCE)
    rc = launch_stage(md, t, u_prev, f, force, 1, H, W, W, (int64_t)W * H, TNRD_STAGE_FORCE, status, s);
    if (rc) return rc;

    train::BwdArgs a;
    a.s = stage_args(md, t, 0u);
    a.H = H; a.W = W; a.m = m; a.kp = md->kp;
    a.u = u_prev; a.f = f; a.force = force; a.g_next = g_next;
    a.g_t = g_t; a.z = z; a.phi = phi; a.dphi = dphi; a.v = v; a.w1 = w1;
    a.adj = g_prev ? adjb : nullptr;
    a.g_prev = g_prev ? g_prev : gp;
    a.part = part;
    a.nblk = nblk;
    a.projected = md->variant == TNRD_VARIANT_PROJECTED;
    a.f0 = 0; a.nf = nfc; a.last_chunk = 0;
    const unsigned pblocks = (unsigned)((n + 255) / 256);
    train::bwd_pointwise_kernel<<<pblocks, 256, 0, s>>>(a);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    if (grad_beta) {
        train::bwd_final_kernel<<<1, 32, 0, s>>>(part, outd, 1, (int)pblocks, 1);  // one warp
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(grad_beta, outd, sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        g_launches.fetch_add(1);
    }
    for (int f0 = 0; f0 < nk; f0 += nfc) {
        a.f0 = f0;
        a.nf = std::min(nfc, nk - f0);
        a.last_chunk = f0 + a.nf >= nk;
        // interior rectangle and border band as separate launches (uniform warps)
        switch (m) {
            case 3: bwd_image_kernels<3>(md, a, H, W, g_prev != nullptr, s); break;
            case 5: bwd_image_kernels<5>(md, a, H, W, g_prev != nullptr, s); break;
            case 7: bwd_image_kernels<7>(md, a, H, W, g_prev != nullptr, s); break;
            default: bwd_image_kernels<9>(md, a, H, W, g_prev != nullptr, s); break;
        }
        CUDA_TRY(cudaGetLastError());
        if (grad_k || grad_w) {
            const size_t rsm = sizeof(float) * (2 * (size_t)m * train::red_row_stride(m) + 4 * train::kSeg);
            const dim3 rgrid((unsigned)nblk, (unsigned)a.nf);
            switch (m) {
                case 3: train::bwd_reduce_kernel<3><<<rgrid, 256, rsm, s>>>(a, nseg); break;
                case 5: train::bwd_reduce_kernel<5><<<rgrid, 256, rsm, s>>>(a, nseg); break;
                case 7: train::bwd_reduce_kernel<7><<<rgrid, 256, rsm, s>>>(a, nseg); break;
                default: train::bwd_reduce_kernel<9><<<rgrid, 256, rsm, s>>>(a, nseg); break;
            }
            const int tot = a.nf * nout;
            train::bwd_final_kernel<<<(tot + 3) / 4, 128, 0, s>>>(part, outd, a.nf, nblk, nout);
            CUDA_TRY(cudaGetLastError());
            g_launches.fetch_add(2);
            std::vector<double> h((size_t)tot);
            CUDA_TRY(cudaMemcpyAsync(h.data(), outd, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            for (int fi = 0; fi < a.nf; ++fi) {
                const double* o = h.data() + (size_t)fi * nout;
                if (grad_k) {
                    double* gk = grad_k + (size_t)(f0 + fi) * mm;
                    // gk = -rot180(C1) - C2 (training.py:108-109)
                    for (int q = 0; q < mm; ++q) gk[q] = -o[mm - 1 - q] - o[mm + q];
                }
                if (grad_w)
                    for (int j = 0; j < M; ++j) grad_w[(size_t)(f0 + fi) * M + j] = -o[2 * mm + j];
            }
        }
    }
    (void)want_params;
    CUDA_TRY(cudaStreamSynchronize(s));
    uint32_t hs[TNRD_STATUS_WORDS];
    CUDA_TRY(cudaMemcpy(hs, status, sizeof hs, cudaMemcpyDeviceToHost));
    int bad = -1;
    return tnrd_status_decode(hs, &bad);
}

// imageops.py:75-106 conv2d_adjoint: exact transpose of conv2d(., k) with the
// half-sample mirror padding, dense H x W device images
extern "C" int tnrd_conv2d_adjoint(const float* img, float* out, int H, int W, const double* k, int m,
                                   void* stream) {
    if (!img || !out || !k) return fail(TNRD_EINVAL, "NULL buffer");
    if (m < 1 || m % 2 != 1) return fail(TNRD_EINVAL, "kernel side must be odd, got %d", m);
    if (m > 15) return fail(TNRD_EUNSUPPORTED, "conv2d_adjoint supports m <= 15, got %d", m);
    if (H < 1 || W < 1) return fail(TNRD_EINVAL, "image must have at least one pixel");
    if (m > 2 * std::min(H, W) + 1)
        return fail(TNRD_EINVAL, "kernel size %d degenerate for image of shape (%d, %d)", m, H, W);
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<float> kf((size_t)m * m);
    for (int i = 0; i < m * m; ++i) {
        if (!std::isfinite(k[i])) return fail(TNRD_EINVAL, "kernel contains non-finite values");
        kf[i] = (float)k[i];
    }
    StreamScratch scr(s);
    float* dk;
    if (scr.get(&dk, kf.size())) return fail(TNRD_ECUDA, "allocation failed");
    CUDA_TRY(cudaMemcpyAsync(dk, kf.data(), kf.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    train::conv2d_adjoint_kernel<<<(unsigned)((H * W + 255) / 256), 256, 0, s>>>(img, out, H, W, dk, m);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    CUDA_TRY(cudaStreamSynchronize(s));  // kf lives on the host stack
    return TNRD_OK;
}

// imageops.py:109-127 patch_correlation: C[a][b] = sum_P pad(base)[P + (a, b)]
// adj[P] (symmetric pad by m/2), dense H x W device images; out: host m x m
// float64.  Synchronous; two-pass fixed-order reduction.
extern "C" int tnrd_patch_correlation(const float* base, const float* adj, int H, int W, int m,
                                      double* out, void* stream) {
    if (!base || !adj || !out) return fail(TNRD_EINVAL, "NULL buffer");
    if (m < 1 || m % 2 != 1) return fail(TNRD_EINVAL, "kernel side must be odd, got %d", m);
    if (H < 1 || W < 1) return fail(TNRD_EINVAL, "image must have at least one pixel");
    if (m > 2 * std::min(H, W) + 1)
        return fail(TNRD_EINVAL, "kernel size %d degenerate for image of shape (%d, %d)", m, H, W);
    cudaStream_t s = (cudaStream_t)stream;
    const int n = H * W, mm = m * m;
    const int nblk = (n + train::kRedPx - 1) / train::kRedPx;
    StreamScratch scr(s);
    double *part, *outd;
    if (scr.get(&part, (size_t)nblk * mm) || scr.get(&outd, mm)) return fail(TNRD_ECUDA, "allocation failed");
    train::patch_corr_kernel<<<nblk, 128, 0, s>>>(base, adj, H, W, m, part);
    train::bwd_final_kernel<<<(mm + 3) / 4, 128, 0, s>>>(part, outd, 1, nblk, mm);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(2);
    CUDA_TRY(cudaMemcpyAsync(out, outd, mm * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return TNRD_OK;
}

// ----------------------------------------------------------------- speckle

// speckle.py:51-70 (statistical parity; tnrd_speckle.cuh)
extern "C" int tnrd_sample_speckle(const float* clean, float* out, int batch, int H, int W,
                                   int64_t ld, int64_t image_stride, int looks, uint64_t seed,
                                   uint32_t* d_status, void* stream) {
    if (!out) return fail(TNRD_EINVAL, "NULL buffer");
    if (looks < 1) return fail(TNRD_EINVAL, "looks must be >= 1, got %d", looks);
    if (batch < 1 || H < 1 || W < 1) return fail(TNRD_EINVAL, "empty image");
    if (ld < W) return fail(TNRD_EINVAL, "row stride %lld < width %d", (long long)ld, W);
    if (batch > 1 && image_stride < ld * H)
        return fail(TNRD_EINVAL, "image stride %lld too small", (long long)image_stride);
    SpeckleArgs a;
    a.clean = clean;
    a.out = out;
    a.ld = ld;
    a.img_stride = image_stride;
    a.H = H; a.W = W; a.batch = batch;
    a.k0 = (uint32_t)seed;
    a.k1 = (uint32_t)(seed >> 32);
    const double d = looks - 1.0 / 3.0;
    a.d = (float)d;
    a.c = (float)(1.0 / std::sqrt(9.0 * d));
    a.inv_l = (float)(1.0 / looks);
    a.status = d_status;
    if (batch > 65535) return fail(TNRD_EINVAL, "batch must be <= 65535");
    dim3 grid((W + 255) / 256, std::min(H, 65535), batch);
    speckle_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    return TNRD_OK;
}

// host restatement of the generator's integer core, for known-answer tests
// (no GPU needed): Philox4x32-10 of (counter, key)
extern "C" void tnrd_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const Philox4 r = philox4x32_10(Philox4{ctr[0], ctr[1], ctr[2], ctr[3]}, key[0], key[1]);
    out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

// ----------------------------------------------------------------- conv2d / prox

struct ConvTaps {
    float k[225];
};

// imageops.py:53-72: out[y,x] = sum_{a,b} k[a,b] img[mir(y+r-a), mir(x+r-b)]
__global__ void conv2d_kernel(const float* __restrict__ img, float* __restrict__ out, int H, int W,
                              int64_t ld, int m, const ConvTaps taps) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= W || y >= H) return;
    const int r = m / 2;
    float s = 0.0f;
    for (int a = 0; a < m; ++a) {
        int yy = y + r - a;
        yy = yy < 0 ? -1 - yy : (yy >= H ? 2 * H - 1 - yy : yy);
        for (int b = 0; b < m; ++b) {
            int xx = x + r - b;
            xx = xx < 0 ? -1 - xx : (xx >= W ? 2 * W - 1 - xx : xx);
            s = fmaf(taps.k[a * m + b], __ldg(img + (int64_t)yy * ld + xx), s);
        }
    }
    out[(int64_t)y * ld + x] = s;
}

extern "C" int tnrd_conv2d(const float* img, float* out, int H, int W, int64_t ld, const double* k,
                           int m, void* stream) {
    if (!img || !out || !k) return fail(TNRD_EINVAL, "NULL buffer");
    if (m < 1 || m % 2 != 1) return fail(TNRD_EINVAL, "kernel side must be odd, got %d", m);
    if (m > 15) return fail(TNRD_EUNSUPPORTED, "conv2d supports m <= 15, got %d", m);
    if (H < 1 || W < 1) return fail(TNRD_EINVAL, "image must have at least one pixel");
    if (m > 2 * std::min(H, W) + 1)
        return fail(TNRD_EINVAL, "kernel size %d degenerate for image of shape (%d, %d)", m, H, W);
    if (ld < W) return fail(TNRD_EINVAL, "row stride too small");
    ConvTaps taps;
    for (int i = 0; i < m * m; ++i) {
        if (!std::isfinite(k[i])) return fail(TNRD_EINVAL, "kernel contains non-finite values");
        taps.k[i] = (float)k[i];
    }
    dim3 blk(32, 8), grid((W + 31) / 32, (H + 7) / 8);
    conv2d_kernel<<<grid, blk, 0, (cudaStream_t)stream>>>(img, out, H, W, ld, m, taps);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    return TNRD_OK;
}

// speckle.py:111-121 (cancellation-free for u~ < 0)
__global__ void prox_kernel(const float* __restrict__ ut, const float* __restrict__ f,
                            float* __restrict__ out, int64_t n, float lam4, float c8, float inv2a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        out[i] = prox_idiv_f(ut[i], f[i], lam4, c8, inv2a);
    }
}

extern "C" int tnrd_prox_idiv(const float* ut, const float* f, float* out, int64_t n, double lam,
                              void* stream) {
    if (!(lam > 0)) return fail(TNRD_EINVAL, "lambda must be positive, got %g", lam);
    if (n <= 0) return TNRD_OK;
    if (!ut || !f || !out) return fail(TNRD_EINVAL, "NULL buffer");
    const double a = 1.0 + 2.0 * lam;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
    prox_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
        ut, f, out, n, (float)(4.0 * lam), (float)(8.0 * a * lam), (float)(1.0 / (2.0 * a)));
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    return TNRD_OK;
}
