/*
 * despeckle_c.c -- the C ABI (include/tnrd.h) used from plain C, without
 * Python or torch: build a random TNRD model the way the reference's tests do
 * (unit-norm zero-mean 7x7 kernels, N(0, 0.1^2) RBF weights on the default
 * 63-centre grid, lambda = 1), despeckle a synthetic speckled image through a
 * plan (host buffers in, host buffers out), and print timing and a checksum.
 *
 *   gcc -O2 -I include examples/despeckle_c.c -L paper_1702_07482_b200 -ltnrd \
 *       -Wl,-rpath,$PWD/paper_1702_07482_b200 -lm -o build/despeckle_c
 *   ./build/despeckle_c [H W]
 *
 * (The zero-mean kernels here are random unit vectors made zero-mean directly;
 * the Python package builds them from the reference's DCT basis.)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "tnrd.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* splitmix64 -> (0, 1) */
    uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return ((z >> 11) + 0.5) / 9007199254740992.0;
}
static double nrand(void) { return sqrt(-2.0 * log(urand())) * cos(6.283185307179586 * urand()); }

static double now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

#define CHECK(x)                                                                 \
    do {                                                                         \
        int rc_ = (x);                                                           \
        if (rc_) {                                                               \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, tnrd_last_error()); \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main(int argc, char** argv) {
    const int H = argc > 2 ? atoi(argv[1]) : 512, W = argc > 2 ? atoi(argv[2]) : 512;
    const int m = 7, nk = 48, T = 5, M = 63;
    const double radius = 310.0, delta = 2.0 * radius / (M - 1), gamma = delta;
    double* k = malloc(sizeof(double) * T * nk * m * m);
    double* w = malloc(sizeof(double) * T * nk * M);
    double lam[5];
    for (int t = 0; t < T; ++t) {
        lam[t] = 1.0;
        for (int i = 0; i < nk; ++i) {
            double* ki = k + ((size_t)t * nk + i) * m * m;
            double mean = 0.0, nrm = 0.0;
            for (int j = 0; j < m * m; ++j) mean += (ki[j] = nrand());
            mean /= m * m;
            for (int j = 0; j < m * m; ++j) {
                ki[j] -= mean;
                nrm += ki[j] * ki[j];
            }
            for (int j = 0; j < m * m; ++j) ki[j] /= sqrt(nrm);
            for (int j = 0; j < M; ++j) w[((size_t)t * nk + i) * M + j] = 0.1 * nrand();
        }
    }
    tnrd_model* model = NULL;
    CHECK(tnrd_model_create(m, nk, T, M, k, w, -radius, delta, gamma, lam, 0, &model));
    tnrd_plan* plan = NULL;
    CHECK(tnrd_plan_create(model, 1, H, W, &plan));
    float* f = malloc(sizeof(float) * H * W);
    float* u = malloc(sizeof(float) * H * W);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const double clean = 40.0 + 150.0 * ((x / 64 + y / 64) % 2);
            const double g = -0.25 * log(urand() * urand() * urand() * urand()); /* Gamma(4, 1/4) */
            f[(size_t)y * W + x] = (float)(clean * sqrt(g));
        }
    CHECK(tnrd_plan_despeckle_host(plan, f, u)); /* warm-up (builds the graph) */
    const int reps = 20;
    const double t0 = now();
    for (int r = 0; r < reps; ++r) CHECK(tnrd_plan_despeckle_host(plan, f, u));
    const double dt = (now() - t0) / reps;
    double sum = 0.0, err_in = 0.0, err_out = 0.0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const double clean = 40.0 + 150.0 * ((x / 64 + y / 64) % 2);
            sum += u[(size_t)y * W + x];
            err_in += fabs(f[(size_t)y * W + x] - clean);
            err_out += fabs(u[(size_t)y * W + x] - clean);
        }
    printf("%s: %dx%d despeckle (7x7, Nk=48, T=5) %.3f ms host-to-host = %.1f MPix/s; "
           "checksum %.6e; mean |f-clean| %.2f -> mean |u-clean| %.2f (random model)\n",
           tnrd_version(), H, W, dt * 1e3, H * W / dt / 1e6, sum, err_in / (H * W),
           err_out / (H * W));
    CHECK(tnrd_plan_destroy(plan));
    CHECK(tnrd_model_destroy(model));
    free(k); free(w); free(f); free(u);
    return 0;
}
