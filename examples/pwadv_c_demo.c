/*
 * pwadv_c_demo.c — the C ABI used from plain C, no Python or torch:
 * generate the BASELINE fields on the device (K5), evaluate the PW advection
 * (K1, device pointers) and through the host-buffer context, and check both
 * bit for bit against the CPU oracle (oracle/pwadv_oracle.c, the test
 * checker). Exit code 0 = identical.
 *
 *   nvcc -o pwadv_c_demo examples/pwadv_c_demo.c oracle/pwadv_oracle.c \
 *        -Iinclude -Lpaper_2010_01545_b200 -lpwadv -Xlinker -rpath=...
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pwadv.h"

/* oracle (test checker) entry points */
void oracle_fill_random(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                        uint64_t seed, int baseline);
void oracle_baseline_coefficients(uint64_t seed, int64_t nz, double *tzc1, double *tzc2,
                                  double *tzd1, double *tzd2);
int oracle_advect(const double *u, const double *v, const double *w, double *su, double *sv,
                  double *sw, int64_t nx, int64_t ny, int64_t nz, double tcx, double tcy,
                  const double *tzc1, const double *tzc2, int engines);

#define CK(x)                                                                        \
    do {                                                                             \
        int rc_ = (x);                                                               \
        if (rc_) {                                                                   \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, pwadv_last_error());    \
            return 2;                                                                \
        }                                                                            \
    } while (0)

int main(int argc, char **argv)
{
    const int64_t nx = argc > 1 ? atoll(argv[1]) : 96, ny = argc > 2 ? atoll(argv[2]) : 80;
    const int64_t nz = argc > 3 ? atoll(argv[3]) : 64;
    const uint64_t seed = 42;
    const size_t n = (size_t)(nx + 2) * (ny + 2) * nz, bytes = n * sizeof(double);
    const double tc = 0.25 / 50.0;
    double *h[9];
    for (int m = 0; m < 9; ++m) h[m] = (double *)calloc(n, sizeof(double));
    double *tz1 = (double *)malloc(nz * sizeof(double)), *tz2 = (double *)malloc(nz * sizeof(double));
    oracle_baseline_coefficients(seed, nz, tz1, tz2, NULL, NULL);

    /* device path: K5 fills, K1 evaluates */
    double *d[6], *dtz;
    for (int m = 0; m < 6; ++m) {
        if (cudaMalloc((void **)&d[m], bytes) != cudaSuccess) return 3;
        cudaMemset(d[m], 0, bytes);
    }
    cudaMalloc((void **)&dtz, 2 * nz * sizeof(double));
    cudaMemcpy(dtz, tz1, nz * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(dtz + nz, tz2, nz * sizeof(double), cudaMemcpyHostToDevice);
    CK(pwadv_fill_f64(d[0], d[1], d[2], nx, ny, nz, 1, seed, 0, 0, 0, NULL));
    CK(pwadv_advect_f64(d[0], d[1], d[2], d[3], d[4], d[5], nx, ny, nz, tc, tc, dtz, dtz + nz,
                        NULL, NULL));
    for (int m = 0; m < 6; ++m) cudaMemcpy(h[m], d[m], bytes, cudaMemcpyDeviceToHost);

    /* oracle on the same inputs */
    double *ref_in[3], *ref_out[3];
    for (int m = 0; m < 3; ++m) {
        ref_in[m] = (double *)malloc(bytes);
        ref_out[m] = (double *)calloc(n, sizeof(double));
    }
    oracle_fill_random(ref_in[0], ref_in[1], ref_in[2], nx, ny, nz, seed, 1);
    oracle_advect(ref_in[0], ref_in[1], ref_in[2], ref_out[0], ref_out[1], ref_out[2], nx, ny, nz,
                  tc, tc, tz1, tz2, 4);
    int bad = 0;
    for (int m = 0; m < 3; ++m) {
        bad |= memcmp(h[m], ref_in[m], bytes) != 0;          /* K5 == reference generator */
        bad |= memcmp(h[3 + m], ref_out[m], bytes) != 0;     /* K1 == oracle, halos included */
    }

    /* host-buffer context (the drop-in entry) on the oracle's inputs */
    pwadv_ctx *ctx = NULL;
    CK(pwadv_ctx_create(&ctx, 0, nx, ny, nz));
    CK(pwadv_ctx_advect_host(ctx, ref_in[0], ref_in[1], ref_in[2], h[6], h[7], h[8], tc, tc, tz1,
                             tz2, 4, NULL));
    for (int m = 0; m < 3; ++m) bad |= memcmp(h[6 + m], ref_out[m], bytes) != 0;
    CK(pwadv_ctx_destroy(ctx));

    printf("pwadv C demo %lldx%lldx%lld: device K5/K1 and host ctx %s the oracle (abi %d)\n",
           (long long)nx, (long long)ny, (long long)nz, bad ? "DIFFER from" : "bit-identical to",
           pwadv_abi_version());
    return bad ? 1 : 0;
}
